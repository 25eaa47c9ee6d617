"""Batched pipelined FP64 GEMM (the DMMA building block of every RSF / peeling step) against a
plain FP64 matmul, including forced split-K with its deterministic workspace reduction.

Bound: |C - C_ref| <= gamma_K (|alpha| |A| |B| + |beta| |C0|) elementwise, gamma_K = 2 K u
(the standard FP64 inner-product error bound with u = 2^-53, doubled for the split sum)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(R, ta, tb, M, N, K, batch, alpha, beta, splitk, seed):
    g = np.random.default_rng(seed)
    A = g.standard_normal((batch, K, M) if ta else (batch, M, K))   # row-major view of column-major op
    B = g.standard_normal((batch, N, K) if tb else (batch, K, N))
    C0 = g.standard_normal((batch, M, N))
    # column-major storage: store the transpose of each row-major matrix
    dev = torch.device('cuda:0')
    dA = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).to(dev)
    dB = torch.from_numpy(np.ascontiguousarray(np.swapaxes(B, 1, 2))).to(dev)
    dC = torch.from_numpy(np.ascontiguousarray(np.swapaxes(C0, 1, 2))).to(dev)
    st = R.lib.rsf_debug_gemm(ta, tb, M, N, K, batch, alpha, dA.data_ptr(), dB.data_ptr(), beta,
                              dC.data_ptr(), splitk)
    assert st == 0
    C = np.swapaxes(dC.cpu().numpy(), 1, 2)
    opA = np.swapaxes(A, 1, 2) if ta else A
    opB = np.swapaxes(B, 1, 2) if tb else B
    ref = alpha * (opA @ opB) + beta * C0
    bound = 2 * max(K, 1) * 2.0 ** -53 * (abs(alpha) * (np.abs(opA) @ np.abs(opB)) + abs(beta) * np.abs(C0)) + 1e-300
    return C, ref, bound


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K,batch", [(1, 1, 1, 1), (130, 70, 33, 3), (257, 31, 2049, 2), (64, 200, 5000, 1),
                                         (7, 300, 40, 5),
                                         # M = 1: the gather-GEMV path (one column tile with K split,
                                         # many tiles, ragged tails, K beyond one shared-memory chunk)
                                         (1, 64, 20000, 1), (1, 200, 5000, 2), (1, 5000, 700, 1), (1, 70, 33, 3),
                                         (1, 131, 9000, 2)])
@pytest.mark.parametrize("splitk", [1, 0, 3, 7])
def test_batched_gemm_vs_matmul(ta, tb, M, N, K, batch, splitk):
    import paper_1603_08057_b200 as R
    C, ref, bound = _run(R, ta, tb, M, N, K, batch, -0.75, 0.5, splitk, seed=M * 131 + N * 7 + K + 3 * ta + tb)
    assert np.all(np.abs(C - ref) <= bound), float(np.max(np.abs(C - ref) / bound))


def test_split_k_is_deterministic():
    import paper_1603_08057_b200 as R
    a = _run(R, 1, 0, 96, 64, 20000, 2, 1.0, 0.0, 5, seed=11)[0]
    b = _run(R, 1, 0, 96, 64, 20000, 2, 1.0, 0.0, 5, seed=11)[0]
    assert np.array_equal(a, b)


def test_empty_and_invalid():
    import paper_1603_08057_b200 as R
    assert R.lib.rsf_debug_gemm(0, 0, 4, 4, 4, 1, 1.0, None, None, 0.0, None, 0) != 0
    t = torch.zeros(16, dtype=torch.float64, device='cuda:0')
    p = t.data_ptr()
    assert R.lib.rsf_debug_gemm(0, 0, 0, 4, 4, 1, 1.0, p, p, 0.0, p, 0) == 0   # M = 0: nothing to do
    # K = 0: C = beta C
    t.fill_(2.0)
    assert R.lib.rsf_debug_gemm(0, 0, 4, 4, 0, 1, 1.0, p, p, 0.5, p, 0) == 0
    assert torch.all(t == 1.0)
