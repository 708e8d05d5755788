"""Config 4 on one B200 (rest_hybrid, 4096 queries, t1+t2+t3): the control
kernel alone (virtual-clock decode, the reference arm's work) and the search
with the real forward on the small and mid model shapes, with the tree-KV
budget (peak live pages) each needs. Prints one JSON line per measurement."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex  # noqa: E402

cfg = (ROOT / "configs" / "c4_rest_w4_q4096.json").read_text()
seed = json.loads(cfg)["run"]["seed"]
ex = spex.Executor(cfg, seed, None, trace=False)
t0 = time.time()
tot = ex.run()
print(json.dumps({"what": "c4 control only", "device_ms": ex.stats()["device_ms"], "wall_s": time.time() - t0,
                  "queries": tot.queries, "makespan_virtual": tot.makespan}), flush=True)
ex.close()
for pol, prm in (("small_policy", "small_prm"), ("mid_policy", "mid_prm")):
    for world in ((1, 2, 4, 8) if pol == "mid_policy" else (1,)):
        for rank in ((0,) if world == 1 else (0, world - 1)):
            ex = spex.Executor(cfg, seed, None, trace=False)
            ex.set_model(pol, prm, weight_seed=1)
            if world > 1:
                ex.set_shard(rank, world)
            t0 = time.time()
            try:
                tot = ex.run()
                ms, kv = ex.model_stats(), ex.kv_stats()
                print(json.dumps({"what": f"c4 {pol}+{prm} rank {rank}/{world}", "step_ms": ms["step_ms"],
                                  "control_ms": ms["control_ms"], "attn_ms": ms["attn_ms"],
                                  "decode_rows": ms["decode_rows"], "prm_rows": ms["prm_rows"],
                                  "queries_per_s_rank": (tot.queries / world) / (ms["step_ms"] / 1000.0),
                                  "kv": kv, "wall_s": time.time() - t0}), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"what": f"c4 {pol}+{prm} rank {rank}/{world}", "error": str(e)}), flush=True)
            ex.close()
