"""Op-level numerics of the sm_100a kernels against plain PyTorch fp32 references."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _gemm(sw, A, B, C, mode):
    M, K = A.shape
    N = B.shape[0]
    sw.check(sw.lib().sw_op_gemm(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                 ctypes.c_void_p(C.data_ptr()), M, N, K, mode, _stream()))
    torch.cuda.synchronize()


def _rel(a, b):
    return float((a - b).float().norm() / b.float().norm().clamp_min(1e-30))


@pytest.mark.parametrize("M", [1, 5, 32, 33, 64, 128, 200, 256, 257, 300, 1000])
@pytest.mark.parametrize("N,K", [(256, 64), (512, 256), (1024, 2048), (3072, 2048)])
def test_gemm_store(swlib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(swlib, A, B, C, 0)
    ref = A.float() @ B.float().T
    assert _rel(C, ref) < 8e-3, (M, N, K)


@pytest.mark.parametrize("M", [3, 64, 129, 512])
def test_gemm_residual(swlib, M):
    K, N = 512, 768 if M <= 256 else 1024
    g = torch.Generator(device="cuda").manual_seed(M)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    _gemm(swlib, A, B, C, 1)
    ref = C0 + A.float() @ B.float().T
    assert _rel(C, ref) < 1e-5 + 4e-3 * float((A.float() @ B.float().T).norm() / ref.norm())


@pytest.mark.parametrize("M,K", [(2, 256), (40, 2048), (256, 256), (300, 512), (64, 4096)])
def test_gemm_swiglu(swlib, M, K):
    F = 512  # 2F rows in [gate 64 | up 64] blocks
    g = torch.Generator(device="cuda").manual_seed(M + 11)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    Wg = (torch.randn(F, K, device="cuda", generator=g) / K ** 0.5)
    Wu = (torch.randn(F, K, device="cuda", generator=g) / K ** 0.5)
    W = torch.empty(2 * F, K, device="cuda")
    for j in range(F // 64):
        W[128 * j:128 * j + 64] = Wg[64 * j:64 * j + 64]
        W[128 * j + 64:128 * j + 128] = Wu[64 * j:64 * j + 64]
    W = W.bfloat16()
    C = torch.zeros(M, F, device="cuda", dtype=torch.bfloat16)
    _gemm(swlib, A, W, C, 2)
    gg = A.float() @ W[0::1].float().T
    gate = torch.cat([gg[:, 128 * j:128 * j + 64] for j in range(F // 64)], 1)
    up = torch.cat([gg[:, 128 * j + 64:128 * j + 128] for j in range(F // 64)], 1)
    ref = torch.nn.functional.silu(gate) * up
    assert _rel(C, ref) < 1e-2


# More feature tiles than SMs at decode widths (the Llama-8B gate/up: 224 tiles): whole tiles per SM
# plus a stream-K remainder with a deterministic partial reduction (gemm_decode2.cu).  Two calls
# back to back also check that the per-tile counters re-arm.
@pytest.mark.parametrize("M", [65, 129, 256])
@pytest.mark.parametrize("N,K", [(28672, 1024), (20480, 2048), (28672, 4096)])
def test_gemm_decode_wide(swlib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ref = A.float() @ B.float().T
    C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(swlib, A, B, C, 0)
    assert _rel(C, ref) < 8e-3, (M, N, K)
    C2 = torch.zeros_like(C)
    _gemm(swlib, A, B, C2, 0)
    assert torch.equal(C, C2)


@pytest.mark.parametrize("M", [129, 256])
def test_gemm_swiglu_wide(swlib, M):
    F, K = 14336, 2048  # 224 tiles of [gate 64 | up 64]
    g = torch.Generator(device="cuda").manual_seed(M + 5)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(2 * F, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    C = torch.zeros(M, F, device="cuda", dtype=torch.bfloat16)
    _gemm(swlib, A, W, C, 2)
    gg = (A.float() @ W.float().T).view(M, F // 64, 2, 64)
    ref = (torch.nn.functional.silu(gg[:, :, 0]) * gg[:, :, 1]).reshape(M, F)
    assert _rel(C, ref) < 1e-2


@pytest.mark.parametrize("rows,dim", [(1, 256), (7, 2048), (300, 4096)])
def test_rmsnorm(swlib, rows, dim):
    x = torch.randn(rows, dim, device="cuda") * 3
    gsc = (1 + 0.1 * torch.randn(dim, device="cuda")).bfloat16()
    y = torch.empty(rows, dim, device="cuda", dtype=torch.bfloat16)
    swlib.check(swlib.lib().sw_op_rmsnorm(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(gsc.data_ptr()),
                                          ctypes.c_void_p(y.data_ptr()), rows, dim, ctypes.c_float(1e-5), _stream()))
    torch.cuda.synchronize()
    ref = x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5) * gsc.float()
    assert _rel(y, ref) < 5e-3
