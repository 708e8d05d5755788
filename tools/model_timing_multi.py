"""Repeated model_timing in one process (warm runs): cfg policy prm reps."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex

name, policy, prm, reps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
cfg = (ROOT / "configs" / f"{name}.json").read_text()
seed = json.loads(cfg)["run"]["seed"]
for r in range(reps):
    ex = spex.Executor(cfg, seed, None, trace=False)
    ex.set_model(policy, prm, weight_seed=1)
    t0 = time.time(); tot = ex.run(); wall = time.time() - t0
    st = ex.stats(); ms = ex.model_stats(); ex.close()
    print(json.dumps({"rep": r, "wall_s": round(wall, 2), "ctl_ms": round(st["device_ms"]), "model_ms": round(ms["model_ms"]),
                      "attn_ms": round(ms["attn_ms"]), "step_ms": round(ms["step_ms"]), "streamed": ms["streamed"]}), flush=True)
