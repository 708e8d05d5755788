"""Microbenchmark: hand-written tcgen05 GEMM (gemm_tc.cu, STORE/LSE epilogues)
vs torch.matmul (cuBLAS) on the same shapes, CUDA-event timed."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from tests.test_gemm_tc_gpu import TcEpilogue, _lib, _maps, EPI_STORE, EPI_LSE  # noqa: E402


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


lib = _lib()
st = torch.cuda.current_stream().cuda_stream
shapes = [(4096, 4096, 4096), (2157, 3072, 1024), (2157, 1024, 1024), (2157, 5632, 1024), (2157, 1024, 2816),
          (2157, 32000, 1024), (8192, 2816, 512)]
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda")
    a, b = _maps(lib, x, w)
    ep = TcEpilogue(kind=EPI_STORE, y=y.data_ptr(), ldy=N, accumulate=0)
    t_tc = bench(lambda: lib.spex_k_gemm_tc(a.ptr, b.ptr, M, N, K, ctypes.byref(ep), st))
    t_cb = bench(lambda: torch.matmul(x, w.T, out=None).float())
    t_cb32 = bench(lambda: torch.mm(x, w.T))
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K}: tc {t_tc * 1e3:.1f} us ({fl / t_tc / 1e9:.0f} TF/s) | cublas bf16-out {t_cb32 * 1e3:.1f} us "
          f"({fl / t_cb32 / 1e9:.0f} TF/s)", flush=True)
