"""Microbenchmark: the hand-written tcgen05 GEMM (gemm_tc.cu) with the epilogue
each projection uses in the model, on the model's shapes, against cuBLAS
(torch.matmul, bf16 out — no epilogue) on the same shapes. Each side is
captured in a CUDA graph and timed by CUDA events around its replay right after
an L2 flush (a 256 MB write): device time, no host launch path; median of `reps`.

  python tools/gemm_bench.py [--shapes mid|named|all] [--sweep]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from tests.test_gemm_tc_gpu import (ROW, TcEpilogue, _lib, _maps, EPI_STORE, EPI_LSE, EPI_SWIGLU,  # noqa: E402
                                    EPI_ROPE_KV)

MODELS = {  # d, H, KVH, dh, F, V, rows per forward (c2 decode step / PRM batch; c5 per GPU)
    "mid_policy": (1024, 8, 8, 128, 2816, 32000, 2157),
    "mid_prm": (512, 4, 4, 128, 1408, 0, 2048),
    "llama3_8b": (4096, 32, 8, 128, 14336, 128256, 975),
    "prm_1p5b": (1536, 12, 2, 128, 8960, 0, 2048),
}


def timed(fn, flush, reps=15):
    """Device time of one launch of `fn` with a cold L2: `fn` is captured in a
    CUDA graph and replayed between events right after an L2 flush, so neither
    side pays its host launch path (Python/ctypes for ours, the ATen dispatch
    for cuBLAS) inside the timed region."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3  # us


def ops(name):
    d, H, KVH, dh, F, V, M = MODELS[name]
    out = [("qkv", M, (H + 2 * KVH) * dh, d, EPI_ROPE_KV), ("o", M, d, H * dh, EPI_STORE),
           ("gate_up", M, 2 * F, d, EPI_SWIGLU), ("down", M, d, F, EPI_STORE)]
    if V:
        out.append(("lm_head", M, V, d, EPI_LSE))
    return out, (H, KVH, dh)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="all")
    ap.add_argument("--sweep", action="store_true", help="also time every tile shape")
    ap.add_argument("--rows", type=int, default=0, help="override M")
    args = ap.parse_args()
    lib = _lib()
    st = torch.cuda.current_stream().cuda_stream
    sched = torch.zeros(2, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    names = {"mid": ["mid_policy", "mid_prm"], "named": ["llama3_8b", "prm_1p5b"]}.get(args.shapes, list(MODELS))
    cg = ctypes.c_int()
    bn = ctypes.c_int()
    for name in names:
        olist, (H, KVH, dh) = ops(name)
        for op, M, N, K, epi in olist:
            M = args.rows or M
            x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            w = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
            a, b = _maps(lib, x, w)
            keep = []
            if epi == EPI_STORE:
                y = torch.zeros(M, N, device="cuda")
                ep = TcEpilogue(kind=EPI_STORE, y=y.data_ptr(), ldy=N, accumulate=1)
            elif epi == EPI_SWIGLU:
                act = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
                ep = TcEpilogue(kind=EPI_SWIGLU, act=act.data_ptr(), F=N // 2)
                keep.append(act)
            elif epi == EPI_LSE:
                part = torch.empty(M, N // 128, 4, device="cuda")
                ep = TcEpilogue(kind=EPI_LSE, part=part.data_ptr(), n_tiles=N // 128, V=N)
                keep.append(part)
            else:
                slots = 4 * M
                rows = np.zeros(M, ROW)
                rows["abs_pos"] = np.arange(M) % 2000
                rows["slot"] = np.arange(M)
                rows_d = torch.from_numpy(rows.view(np.uint8).copy()).cuda()
                rope = torch.rand(M, dh, device="cuda")
                Qr = torch.empty(M, H, dh, device="cuda")
                Kp = torch.empty(KVH, slots, dh, dtype=torch.bfloat16, device="cuda")
                Vp = torch.empty(KVH, slots, dh, dtype=torch.bfloat16, device="cuda")
                keep += [rows_d, rope, Qr, Kp, Vp]
                ep = TcEpilogue(kind=EPI_ROPE_KV, rows=rows_d.data_ptr(), rope=rope.data_ptr(), H=H, KVH=KVH, dh=dh,
                                qscale=dh ** -0.5, Qr=Qr.data_ptr(), Kp=Kp.data_ptr(), Vp=Vp.data_ptr(), slots=slots)
            fl = 2.0 * M * N * K
            lib.spex_k_gemm_tc_shape(M, N, K, epi, ctypes.byref(cg), ctypes.byref(bn))
            res = {"model": name, "op": op, "M": M, "N": N, "K": K, "auto": [cg.value, bn.value]}

            def run(c=0, n=0):
                rc = lib.spex_k_gemm_tc_ex(a.ptr, b.ptr, M, N, K, ctypes.byref(ep), sched.data_ptr(), c, n,
                                           torch.cuda.current_stream().cuda_stream)
                assert rc == 0, rc

            t = timed(run, flush)
            res["tc_us"] = round(t, 2)
            res["tc_tflops"] = round(fl / t / 1e6, 1)
            tcb = timed(lambda: torch.mm(x, w.T), flush)
            res["cublas_bf16_us"] = round(tcb, 2)
            res["cublas_tflops"] = round(fl / tcb / 1e6, 1)
            res["tc_over_cublas"] = round(tcb / t, 3)
            if args.sweep:
                for c, n in [(2, 256), (2, 128), (1, 256), (1, 128)] + ([(1, 64)] if epi == EPI_STORE else []):
                    res[f"tc_{c}x{n}_us"] = round(timed(lambda: run(c, n), flush), 2)
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
