"""GEMM milestone timing (probe build, lib/probe/libspex_probe.so): per CTA
globaltimer stamps at entry, after griddepcontrol.wait, first TMA issue, first
stage landed, first tile's MMAs issued, epilogue start of tiles 0-2, epilogue
end and exit. Prints per shape / tile config the medians over CTAs (us,
relative to the earliest CTA entry)."""
import ctypes
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ["SPEX_LIB_PATH"] = str(ROOT / "paper_2605_10195_b200" / "lib" / "probe" / "libspex_probe.so")
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from tests.test_gemm_tc_gpu import TcEpilogue, _lib, _maps, EPI_STORE, EPI_SWIGLU  # noqa: E402

lib = _lib()
lib.spex_gemm_probe_set.argtypes = [ctypes.c_void_p]
st = torch.cuda.current_stream().cuda_stream
sched = torch.zeros(2, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
dbg = torch.zeros(296 * 16, dtype=torch.int64, device="cuda")
lib.spex_gemm_probe_set(dbg.data_ptr())
NAMES = {0: "entry", 1: "pdl_wait", 2: "tma0", 3: "stage0", 4: "mma_t0", 5: "epi_t0", 7: "epi_t1", 9: "epi_t2",
         10: "mma_t1", 11: "epi_end", 12: "exit"}
for (name, M, N, K, epi) in [("mid o", 2157, 1024, 1024, EPI_STORE), ("mid down", 2157, 1024, 2816, EPI_STORE),
                             ("mid gate_up", 2157, 5632, 1024, EPI_SWIGLU), ("8b o", 975, 4096, 4096, EPI_STORE)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    a, b = _maps(lib, x, w)
    keep = []
    if epi == EPI_STORE:
        y = torch.zeros(M, N, device="cuda")
        ep = TcEpilogue(kind=EPI_STORE, y=y.data_ptr(), ldy=N, accumulate=1)
    else:
        act = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
        ep = TcEpilogue(kind=EPI_SWIGLU, act=act.data_ptr(), F=N // 2)
        keep.append(act)
    for cg, bn in ((2, 128), (1, 128), (2, 256)):
        for rep in range(4):
            flush.zero_()
            dbg.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            rc = lib.spex_k_gemm_tc_ex(a.ptr, b.ptr, M, N, K, ctypes.byref(ep), sched.data_ptr(), cg, bn, st)
            ev1.record()
            torch.cuda.synchronize()
            assert rc == 0
        # back-to-back: the marginal device time of a second identical launch
        flush.zero_()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        lib.spex_k_gemm_tc_ex(a.ptr, b.ptr, M, N, K, ctypes.byref(ep), sched.data_ptr(), cg, bn, st)
        e1.record()
        lib.spex_k_gemm_tc_ex(a.ptr, b.ptr, M, N, K, ctypes.byref(ep), sched.data_ptr(), cg, bn, st)
        e2.record()
        torch.cuda.synchronize()
        b2b = (e0.elapsed_time(e1) * 1e3, e1.elapsed_time(e2) * 1e3)
        d = dbg.view(296, 16).cpu().numpy().astype(np.int64)
        live = d[:, 0] > 0
        d = d[live]
        t0 = d[:, 0].min()
        res = {"shape": name, "cg": cg, "bn": bn, "ctas": int(live.sum()), "event_us": round(ev0.elapsed_time(ev1) * 1e3, 2),
               "span_us": round((d[:, 12].max() - t0) / 1e3, 2),
               "first_us": round(b2b[0], 2), "second_us": round(b2b[1], 2)}
        for k, nm in NAMES.items():
            col = d[:, k]
            col = col[col > 0]
            if len(col):
                res[nm] = round(float(np.median(col - t0)) / 1e3, 2)
        print(json.dumps(res), flush=True)
