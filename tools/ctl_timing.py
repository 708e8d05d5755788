"""Times the device control kernel per config (CUDA events) next to the reference CPU run."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex
from tests import refutil

names = sys.argv[1:] or ["c1_rebase_w4_q16", "c2_rebase_w16_q256", "c3_rstar_w4_q512", "c5_rebase_w32_q64"]
for n in names:
    cfg = (ROOT / "configs" / f"{n}.json").read_text()
    seed = json.loads(cfg)["run"]["seed"]
    for trace in (1, 0):
        ex = spex.Executor(cfg, seed, None, trace=bool(trace))
        t0 = time.time(); tot = ex.run(); wall = time.time() - t0
        st = ex.stats(); ex.close()
        print(json.dumps({"cfg": n, "trace": trace, "wall_s": round(wall, 4), "device_ms": round(st["device_ms"], 3),
                          "iterations": st["iterations"], "epochs": st["epochs"], "rewards": st["reward_events"],
                          "nodes": st["nodes"], "queries": tot.queries, "makespan": tot.makespan}), flush=True)
    if refutil.ref_lib() is not None:
        import ctypes
        L = refutil.ref_lib(); secs = ctypes.c_double(); tot = (ctypes.c_double * 24)()
        L.ref_run_timed(cfg.encode(), seed, None, 0, 1, ctypes.byref(secs), tot)
        print(json.dumps({"cfg": n, "reference_cpu_s": secs.value, "makespan": tot[0]}), flush=True)
