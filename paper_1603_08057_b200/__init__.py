"""B200-native GP likelihood engine: l(theta), g(theta) via RSF + weak peeling.

Thin Python binding over librsf.so (include/rsf.h).  Every step of the path
runs in the CUDA library; this module only marshals arguments.  Arrays may be
torch tensors (CUDA or CPU) or numpy arrays (host); they must be float64 and
contiguous.  PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field

from . import _lib
from ._lib import FAMILY, PARAM, rsf_eval_diag, rsf_fact_diag, rsf_kernel, rsf_opts, rsf_peel_diag

__all__ = ["Context", "Kernel", "Opts", "Factor", "peel_trace", "gp_mle_eval", "RsfError", "lib",
           "kernel_launches", "nccl_unique_id", "nccl_calls", "col_slice"]

lib = _lib.load()


class RsfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rsf status {code}: {msg}")
        self.code = code


def _check(st):
    if st != 0:
        raise RsfError(st, lib.rsf_last_error().decode())


def kernel_launches() -> int:
    return int(lib.rsf_kernel_launches())


def _order_after_caller(ctx_h):
    """Stream ordering (include/rsf.h conventions): the library's context stream waits for the
    work torch has enqueued so far on its current stream (inputs produced there, outputs
    cloned there).  The library returns only after its own work is complete."""
    torch = sys.modules.get("torch")
    if torch is None or not torch.cuda.is_available() or not torch.cuda.is_initialized():
        return
    _check(lib.rsf_ctx_wait_stream(ctx_h, C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def _ptr(a, dtype_ok=True):
    """(address, keepalive) of a float64 contiguous torch tensor or numpy array."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise TypeError("tensors must be contiguous float64")
            return a.data_ptr(), a
    except ImportError:  # pragma: no cover
        pass
    import numpy as np
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise TypeError("arrays must be C-contiguous float64")
        return a.ctypes.data, a
    raise TypeError(f"unsupported array type {type(a)}")


@dataclass
class Kernel:
    family: str
    rho: float
    sigma2: float = 1.0
    nugget: float = 0.0
    alpha: float = 1.0
    theta: tuple = ("rho",)
    rho2: float = 0.0      # > 0: anisotropic lengths (rho, rho2)

    def c(self) -> rsf_kernel:
        k = rsf_kernel()
        k.family = FAMILY[self.family]
        k.rho, k.sigma2, k.nugget, k.alpha = self.rho, self.sigma2, self.nugget, self.alpha
        k.rho2 = self.rho2
        k.p = len(self.theta)
        for i, t in enumerate(self.theta):
            k.theta[i] = PARAM[t]
        return k


@dataclass
class Opts:
    eps_peel: float = 1e-6
    oversample: int = 8
    probe_block: int = 512
    peel_start: int = 64
    max_depth: int = 30
    r_near: float = 1.8
    r_in: float = 1.75
    r_out: float = 2.45
    seed: int = 1603080570
    strong: int = 0        # 1: strong-admissibility peeling (perfect quadtrees)
    peel_f32: int = 0      # 1: peeled levels stored in FP32, FP64 arithmetic

    def c(self) -> rsf_opts:
        o = rsf_opts()
        for f, _ in rsf_opts._fields_:
            setattr(o, f, getattr(self, f))
        return o


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for rsf_ctx_create_group (rank 0 calls it, then distributes it)."""
    buf = (C.c_ubyte * 128)()
    _check(lib.rsf_nccl_unique_id(buf))
    return bytes(buf)


def nccl_calls() -> int:
    """NCCL collectives this process has issued so far (include/rsf.h; tests)."""
    return int(lib.rsf_debug_nccl_calls())


def col_slice(k: int, parts: int, part: int):
    """[lo, hi) of the probe columns part `part` of `parts` owns (include/rsf.h)."""
    lo, hi = C.c_int64(), C.c_int64()
    lib.rsf_debug_col_slice(k, parts, part, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def group_id_from_process_group():
    """(id_bytes, rank, world) for Context(group=...): rank 0 draws the NCCL unique id and the
    default torch.distributed group broadcasts it (any backend; plumbing only)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    return obj[0], rank, world


class Context:
    """rsf_ctx.  group=(id_bytes, rank, world): one rank of a sharded group (NCCL);
    nccl_comm: an existing ncclComm_t address of the caller instead."""

    def __init__(self, device: int = 0, stream=None, group=None, nccl_comm=None):
        h = C.c_void_p()
        s = None
        if stream is not None:
            s = C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        if group is not None:
            uid, rank, world = group
            buf = (C.c_ubyte * 128).from_buffer_copy(bytes(uid))
            _check(lib.rsf_ctx_create_group(device, s, buf, int(rank), int(world), C.byref(h)))
        else:
            _check(lib.rsf_ctx_create(device, s, C.c_void_p(nccl_comm) if nccl_comm else None, C.byref(h)))
        self.h = h

    @classmethod
    def from_process_group(cls, device: int, stream=None):
        """Collective over the default torch.distributed group (plumbing only): rank 0 draws
        the NCCL id, torch.distributed broadcasts it, every rank joins the group."""
        return cls(device, stream, group=group_id_from_process_group())

    def group(self):
        r, w = C.c_int(), C.c_int()
        _check(lib.rsf_ctx_group(self.h, C.byref(r), C.byref(w)))
        return r.value, w.value

    def close(self):
        if self.h:
            lib.rsf_ctx_destroy(self.h)
            self.h = None

    def __del__(self, _finalizing=sys.is_finalizing):
        if _finalizing():   # process exit: the driver reclaims everything; CUDA may be torn down
            return
        try:
            self.close()
        except Exception:
            pass


class Factor:
    """rsf_factor: which=None -> F ~ Sigma; which=i -> apply-only compression of Sigma_i."""

    def __init__(self, ctx: Context, xy, kernel: Kernel, eps: float, leaf: int = 64,
                 which: int | None = None, opts: Opts | None = None):
        p, keep = _ptr(xy)
        n = (xy.shape[0])
        h = C.c_void_p()
        kc = kernel.c()
        oc = (opts or Opts()).c()
        _order_after_caller(ctx.h)
        _check(lib.rsf_factor(ctx.h, p, n, C.byref(kc), -1 if which is None else which, eps, leaf,
                              C.byref(oc), C.byref(h)))
        self.h, self.ctx, self.n, self.which = h, ctx, n, which

    def close(self):
        if self.h:
            lib.rsf_fact_destroy(self.h)
            self.h = None

    def __del__(self, _finalizing=sys.is_finalizing):
        if _finalizing():   # process exit: the driver reclaims everything; CUDA may be torn down
            return
        try:
            self.close()
        except Exception:
            pass

    def logdet(self) -> float:
        v = C.c_double()
        _check(lib.rsf_logdet(self.h, C.byref(v)))
        return v.value

    def info(self) -> rsf_fact_diag:
        d = rsf_fact_diag()
        _check(lib.rsf_fact_info(self.h, C.byref(d)))
        return d

    def _op(self, fn, b, out):
        pb, kb = _ptr(b)
        po, ko = _ptr(out)
        nrhs = 1 if b.ndim == 1 else b.shape[0]
        # (nrhs, n) row-major == column-major n x nrhs with ld = n
        _order_after_caller(self.ctx.h)
        _check(fn(self.h, pb, po, nrhs, self.n))
        return out

    def solve(self, b, out=None):
        """x = F^-1 b; b is (n,) or (nrhs, n) (each row a right-hand side)."""
        out = b.clone() if out is None and hasattr(b, "clone") else (b.copy() if out is None else out)
        return self._op(lib.rsf_solve, b, out)

    def apply(self, x, out=None):
        out = x.clone() if out is None and hasattr(x, "clone") else (x.copy() if out is None else out)
        return self._op(lib.rsf_apply, x, out)

    def sample(self, w, out=None):
        out = w.clone() if out is None and hasattr(w, "clone") else (w.copy() if out is None else out)
        return self._op(lib.rsf_sample, w, out)


def peel_trace(F: Factor, Fi: Factor | None, eps_peel: float = 1e-6, opts: Opts | None = None,
               trace_id: int = 0):
    v = C.c_double()
    d = rsf_peel_diag()
    oc = (opts or Opts()).c()
    _check(lib.peel_trace(F.h, Fi.h if Fi is not None else None, eps_peel, C.byref(oc), trace_id,
                          C.byref(v), C.byref(d)))
    return v.value, d


def gp_profile_eval(ctx: Context, xy, z, kernel: Kernel, eps: float, leaf: int = 64,
                    opts: Opts | None = None) -> "EvalResult":
    """Log profile likelihood (Eq. prof) and gradient; diag.quad = z^T (Sigma + 1 1^T)^-1 z."""
    px, kx = _ptr(xy)
    pz, kz = _ptr(z)
    n = xy.shape[0]
    kc = kernel.c()
    oc = (opts or Opts()).c()
    ell = C.c_double()
    grad = (C.c_double * 4)()
    d = rsf_eval_diag()
    _order_after_caller(ctx.h)
    _check(lib.gp_profile_eval(ctx.h, px, pz, n, C.byref(kc), eps, leaf, C.byref(oc), C.byref(ell), grad,
                               C.byref(d)))
    return EvalResult(ell.value, [grad[i] for i in range(len(kernel.theta))], d)


def gp_cond_mean(F: Factor, z, xy_new, out=None):
    """Kriging mean Sigma_12 F^-1 z at the rows of xy_new (m x 2)."""
    import torch
    m = xy_new.shape[0]
    if out is None:
        out = torch.empty(m, dtype=torch.float64, device=xy_new.device) if hasattr(xy_new, "device") else \
            __import__("numpy").empty(m)
    pz, kz = _ptr(z)
    px, kx = _ptr(xy_new)
    po, ko = _ptr(out)
    _order_after_caller(F.ctx.h)
    _check(lib.gp_cond_mean(F.h, pz, px, m, po))
    return out


def gp_cond_sample(F: Factor, F22: Factor, z, w, out=None):
    """Conditional samples (Remark conditional).  F: full factor of the joint points
    [x_new; x_data] (new first), F22: factor of the data points, z: (n2,) data values, w:
    (nrhs, m + n2) standard normal rows -> (nrhs, m) samples of z' | z."""
    m = F.n - F22.n
    nrhs = 1 if w.ndim == 1 else w.shape[0]
    if out is None:
        if hasattr(w, "new_empty"):
            out = w.new_empty((nrhs, m)) if w.ndim > 1 else w.new_empty((m,))
        else:
            out = __import__("numpy").empty((nrhs, m) if w.ndim > 1 else (m,))
    pz, kz = _ptr(z)
    pw, kw = _ptr(w)
    po, ko = _ptr(out)
    _order_after_caller(F.ctx.h)
    _check(lib.gp_cond_sample(F.h, F22.h, m, pz, pw, po, nrhs))
    return out


def hutch_trace(F: Factor, Fi: Factor | None, nprobe: int = 64, seed: int = 1603080570):
    """Hutchinson estimate of Tr(F^-1 F_i) (Fi None: Tr(F^-1)) -> (trace, standard error)."""
    t = C.c_double()
    se = C.c_double()
    _check(lib.hutch_trace(F.h, Fi.h if Fi is not None else None, nprobe, seed, C.byref(t), C.byref(se)))
    return t.value, se.value


@dataclass
class EvalResult:
    ell: float
    grad: list
    diag: rsf_eval_diag = field(repr=False)


def gp_mle_eval(ctx: Context, xy, z, kernel: Kernel, eps: float, leaf: int = 64,
                opts: Opts | None = None) -> EvalResult:
    px, kx = _ptr(xy)
    pz, kz = _ptr(z)
    n = xy.shape[0]
    kc = kernel.c()
    oc = (opts or Opts()).c()
    ell = C.c_double()
    grad = (C.c_double * 4)()
    d = rsf_eval_diag()
    _order_after_caller(ctx.h)
    _check(lib.gp_mle_eval(ctx.h, px, pz, n, C.byref(kc), eps, leaf, C.byref(oc), C.byref(ell), grad,
                           C.byref(d)))
    return EvalResult(ell.value, [grad[i] for i in range(len(kernel.theta))], d)
