"""Split mode per-rank step times on ONE B200 (Executor.emulate_split): for
each W, every rank of the job runs in turn with its model while the other
ranks' control runs beside it; the W-GPU step is the max over ranks (the
exchange is timing-independent, so each rank's work is the multi-GPU run's).
Usage: python tools/split_scaling.py CONFIG POLICY PRM W [W ...]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex  # noqa: E402


def rank_run(cfg, seed, policy, prm, rank, world):
    ex = spex.Executor(cfg, seed, None, trace=False)
    ex.set_model(policy, prm, 1)
    if world > 1:
        ex.emulate_split(rank, world)
    t = ex.run()
    m, st = ex.model_stats(), ex.stats()
    out = {"rank": rank, "world": world, "queries": t.queries, "step_ms": m["step_ms"], "control_ms": st["device_ms"],
           "attn_ms": m["attn_ms"], "decode_rows": m["decode_rows"], "prm_rows": m["prm_rows"],
           "makespan_virtual": t.makespan, **ex.split_stats(), "kv": ex.kv_stats()}
    ex.close()
    return out


def main():
    name, policy, prm = sys.argv[1:4]
    cfg = (ROOT / "configs" / f"{name}.json").read_text()
    seed = json.loads(cfg)["run"]["seed"]
    for w in [int(x) for x in sys.argv[4:]]:
        rows = []
        for r in range(w):
            try:
                rank_run(cfg, seed, policy, prm, r, w) if r == 0 else None  # warm-up (shapes, pools)
                rows.append(rank_run(cfg, seed, policy, prm, r, w))
            except Exception as e:  # noqa: BLE001
                rows.append({"rank": r, "world": w, "error": str(e)[:300]})
            print(json.dumps({"what": f"{name} {policy}+{prm} split rank {r}/{w}", **rows[-1]}), flush=True)
        ok = [x for x in rows if "error" not in x]
        if len(ok) == w:
            step = max(x["step_ms"] for x in ok)
            q = sum(x["queries"] for x in ok)
            print(json.dumps({"what": f"{name} split W={w}", "step_ms_max": step, "queries": q,
                              "queries_per_s": q / (step / 1000.0),
                              "control_ms_max": max(x["control_ms"] for x in ok),
                              "xch_rounds": [x["rounds"] for x in ok],
                              "xch_wait_ms_max": max(x["wait_ms"] for x in ok)}), flush=True)


if __name__ == "__main__":
    main()
