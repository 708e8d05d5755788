"""Coupled-mode (one search, control replicated, model work by query block)
per-rank step times for W = 1, 2, 4, 8, measured on ONE GPU by running every
rank of W in turn (each rank's work is exactly what it would run on its own
B200: the whole control kernel plus its block's forward). The W-GPU step is
the max over ranks; this is a per-rank measurement, not a multi-GPU run.

usage: python tools/coupled_scaling.py [config] [policy] [prm] [worlds]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import paper_2605_10195_b200 as spex
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2_rebase_w16_q256"
    policy = sys.argv[2] if len(sys.argv) > 2 else "mid_policy"
    prm = sys.argv[3] if len(sys.argv) > 3 else "mid_prm"
    worlds = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "1,2,4,8").split(",")]
    cfg = (ROOT / "configs" / f"{cfg_name}.json").read_text()
    seed = json.loads(cfg)["run"]["seed"]
    Q = json.loads(cfg)["run"]["n_queries"]

    def search(rank, world):
        ex = spex.Executor(cfg, seed, None, trace=False)
        ex.set_model(policy, prm, weight_seed=1)
        ex.set_shard(rank, world)
        ex.run()
        st, ms = ex.stats(), ex.model_stats()
        ex.close()
        return {"rank": rank, "step_ms": ms["step_ms"], "control_ms": st["device_ms"], "model_ms": ms["model_ms"],
                "attn_ms": ms["attn_ms"], "decode_rows": ms["decode_rows"], "prm_rows": ms["prm_rows"],
                "streamed": ms["streamed"]}

    search(0, 1)  # warm-up
    out = []
    for w in worlds:
        ranks = [search(r, w) for r in range(w)]
        step = max(r["step_ms"] for r in ranks)
        rec = {"config": cfg_name, "policy": policy, "prm": prm, "world": w, "queries": Q,
               "step_ms_max_over_ranks": step, "queries_per_s": Q / (step / 1000.0), "ranks": ranks}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    base = out[0]["queries_per_s"]
    print(json.dumps({"strong_scaling_efficiency": {r["world"]: r["queries_per_s"] / base / r["world"] for r in out}}))


if __name__ == "__main__":
    main()
