"""Tensor-core building blocks (skan_tc.cuh): tcgen05 kind::tf32 MMA from
canonical K-major shared-memory tiles, TMEM accumulation and readback,
checked against an f64 numpy GEMM.  3xTF32 must reach ~1e-6 relative (the
fast path's 1e-5 bar with margin); a single tf32 pass cannot."""
import numpy as np
import pytest

from paper_2512_15742_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ts", [0, 200, 300], ids=["smem_a", "tmem_a", "tmem_a_cp"])
@pytest.mark.parametrize("n,k", [(16, 8), (64, 32), (256, 64), (208, 40)])
def test_tf32x3_gemm_matches_f64(n, k, ts):
    """ts = 200: A written to TMEM with tcgen05.st and read by the MMA from
    there; ts = 300: A staged in shared memory and moved to TMEM by
    tcgen05.cp (the layer GEMM's form).  The tensor core truncates a TMEM
    operand to tf32 the same way, so the lo terms still carry the rest."""
    import torch
    rng = np.random.default_rng(n + k)
    a = rng.standard_normal((128, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = {}
    for passes in (1, 3):
        dd = torch.zeros((128, n), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().skan_debug_gemm_tf32(da.data_ptr(), db.data_ptr(), dd.data_ptr(), n, k, passes + ts,
                                                   torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        out[passes] = np.max(np.abs(dd.cpu().numpy() - want) / scale)
    assert out[3] < 2e-6, out
    assert out[1] > 1e-5, out  # one tf32 pass really is coarser (the test sees the lo terms)


@pytest.mark.parametrize("n,k", [(16, 16), (128, 32), (256, 64), (208, 48)])
def test_f16_ss_gemm_matches_fp16_rounded_inputs(n, k):
    """kind::f16 with both operands in shared memory (the layer GEMM's fp16
    split-precision form): D = fp16(A) fp16(B) accumulated in f32, checked
    against the f64 product of the fp16-rounded inputs."""
    import torch
    rng = np.random.default_rng(7 * n + k)
    a = rng.standard_normal((128, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    a16, b16 = a.astype(np.float16).astype(np.float64), b.astype(np.float16).astype(np.float64)
    want = a16 @ b16
    scale = np.abs(a16) @ np.abs(b16)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dd = torch.zeros((128, n), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().skan_debug_gemm_tf32(da.data_ptr(), db.data_ptr(), dd.data_ptr(), n, k, 1000,
                                               torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert np.max(np.abs(dd.cpu().numpy() - want) / scale) < 1e-6
