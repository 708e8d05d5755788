"""Control kernel + policy/PRM forward timing for one config (GPU)."""
import json, os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex

name = sys.argv[1]; policy = sys.argv[2]; prm = sys.argv[3] if len(sys.argv) > 3 else ""
cfg = (ROOT / "configs" / f"{name}.json").read_text()
seed = json.loads(cfg)["run"]["seed"]
ex = spex.Executor(cfg, seed, None, trace=False)
ex.set_model(policy, prm, weight_seed=1)
t0 = time.time(); tot = ex.run(); wall = time.time() - t0
st = ex.stats(); ms = ex.model_stats(); ex.close()
print(json.dumps({"cfg": name, "policy": policy, "prm": prm, "wall_s": wall, "ctl_ms": st["device_ms"],
                  "queries": tot.queries, **ms}), flush=True)
