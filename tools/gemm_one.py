"""Runs one tcgen05 GEMM configuration `--reps` times (for ncu captures):
  python tools/gemm_one.py --model llama3_8b --op gate_up --cg 2 --bn 256
"""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from tools import gemm_bench as gb  # noqa: E402
from tests.test_gemm_tc_gpu import TcEpilogue, _lib, _maps, EPI_STORE, EPI_SWIGLU, EPI_LSE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3_8b")
ap.add_argument("--op", default="gate_up")
ap.add_argument("--cg", type=int, default=0)
ap.add_argument("--bn", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--rows", type=int, default=0)
a = ap.parse_args()
lib = _lib()
olist, (H, KVH, dh) = gb.ops(a.model)
op, M, N, K, epi = [o for o in olist if o[0] == a.op][0]
M = a.rows or M
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
ma, mb = _maps(lib, x, w)
if epi == EPI_STORE:
    y = torch.zeros(M, N, device="cuda")
    ep = TcEpilogue(kind=EPI_STORE, y=y.data_ptr(), ldy=N, accumulate=1)
elif epi == EPI_SWIGLU:
    y = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
    ep = TcEpilogue(kind=EPI_SWIGLU, act=y.data_ptr(), F=N // 2)
else:
    y = torch.empty(M, N // 128, 4, device="cuda")
    ep = TcEpilogue(kind=EPI_LSE, part=y.data_ptr(), n_tiles=N // 128, V=N)
sched = torch.zeros(2, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    assert lib.spex_k_gemm_tc_ex(ma.ptr, mb.ptr, M, N, K, ctypes.byref(ep), sched.data_ptr(), a.cg, a.bn, st) == 0
torch.cuda.synchronize()
print("ok", M, N, K)
