"""C-ABI checks that need no GPU: the library loads, exports every function
include/rsf.h declares, the ctypes structs match the C layout, and argument
validation fails loudly (RSF_EINVAL) without touching a device."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsf.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:rsf_status|void|const char\*|int64_t)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1603_08057_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import importlib.util
        spec = importlib.util.spec_from_file_location("rsfbuild", os.path.join(ROOT, "paper_1603_08057_b200", "build.py"))
        m = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(m)
        m.build()
    return _lib.load()


def test_header_declares_the_boundary():
    names = _declared_functions()
    for f in ("rsf_factor", "rsf_logdet", "rsf_solve", "rsf_apply", "rsf_sample", "peel_trace", "gp_mle_eval"):
        assert f in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1603_08057_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [f for f in _declared_functions() if f not in exported]
    assert not missing, missing
    for f in _declared_functions():
        getattr(lib, f)


def test_ctypes_struct_layout_matches_c():
    """Compile a C probe against include/rsf.h and compare sizeof/offsetof with ctypes."""
    from paper_1603_08057_b200 import _lib
    structs = {"rsf_kernel": _lib.rsf_kernel, "rsf_opts": _lib.rsf_opts, "rsf_fact_diag": _lib.rsf_fact_diag,
               "rsf_peel_diag": _lib.rsf_peel_diag, "rsf_eval_diag": _lib.rsf_eval_diag}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for nm, st in structs.items():
        lines.append(f'printf("{nm} %zu\\n", sizeof({nm}));')
        for f, _ in st._fields_:
            lines.append(f'printf("{nm}.{f} %zu\\n", offsetof({nm}, {f}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        cf = os.path.join(d, "p.c")
        open(cf, "w").write("\n".join(lines))
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-std=c99", "-o", exe, cf], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = dict(ln.rsplit(" ", 1) for ln in out.strip().splitlines())
    for nm, st in structs.items():
        assert int(got[nm]) == C.sizeof(st), nm
        for f, _ in st._fields_:
            assert int(got[f"{nm}.{f}"]) == getattr(st, f).offset, (nm, f)


def test_null_arguments_are_einval_without_a_device(lib):
    from paper_1603_08057_b200 import _lib
    k = _lib.rsf_kernel()
    k.family, k.rho, k.sigma2, k.nugget, k.alpha, k.p = 0, 0.1, 1.0, 0.01, 1.0, 1
    h = C.c_void_p()
    assert lib.rsf_factor(None, None, 10, C.byref(k), -1, 1e-8, 64, None, C.byref(h)) == _lib.RSF_EINVAL
    assert lib.rsf_last_error()
    ell = C.c_double()
    assert lib.gp_mle_eval(None, None, None, 10, C.byref(k), 1e-8, 64, None, C.byref(ell), None, None) == _lib.RSF_EINVAL
    v = C.c_double()
    assert lib.rsf_logdet(None, C.byref(v)) == _lib.RSF_EINVAL
    assert lib.peel_trace(None, None, 1e-6, None, 0, C.byref(v), None) == _lib.RSF_EINVAL


def test_opts_defaults(lib):
    from paper_1603_08057_b200 import _lib
    o = _lib.rsf_opts()
    lib.rsf_opts_default(C.byref(o))
    assert o.eps_peel == 1e-6 and o.oversample == 8 and o.r_near == 1.8 and o.r_in == 1.75 and o.r_out == 2.45


def test_package_has_no_cpu_fallback():
    """The binding only marshals: no numpy/torch arithmetic of the method, no oracle import."""
    src = open(os.path.join(ROOT, "paper_1603_08057_b200", "__init__.py")).read()
    assert "oracle" not in src
    for bad in ("np.linalg", "torch.linalg", "cholesky", "scipy"):
        assert bad not in src
