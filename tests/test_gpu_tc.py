"""tcgen05 / TMEM / TMA-tensor GEMM plumbing (prefill path f4) vs torch, on the GPU."""
import ctypes

import numpy as np
import pytest

import paper_2512_16473_b200 as moe

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 384, 512), (200, 136, 4096), (1024, 1024, 1024)])
def test_tc_gemm_plain_matches_torch(M, N, K):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    f = moe.lib().moe_debug_tc_gemm
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                  ctypes.c_void_p]
    f.restype = ctypes.c_int
    assert f(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T
    err = (C.double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
