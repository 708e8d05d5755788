"""Control-kernel phase cycles (SPEX_PHASES) of one c2 search solo (no model)
and under load (policy + PRM forward streaming beside it)."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["SPEX_PHASES"] = "1"
import paper_2605_10195_b200 as spex  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rebase_w16_q256"
cfg = (ROOT / "configs" / f"{name}.json").read_text()
seed = json.loads(cfg)["run"]["seed"]
for label, model in (("solo", None), ("solo", None), ("load", ("mid_policy", "mid_prm")),
                     ("load", ("mid_policy", "mid_prm")), ("load_noprm", ("mid_policy", ""))):
    ex = spex.Executor(cfg, seed, None, trace=False)
    if model:
        ex.set_model(model[0], model[1], weight_seed=1)
    ex.run()
    st = ex.stats()
    ms = ex.model_stats() if model else {}
    ex.close()
    print(json.dumps({"label": label, "control_ms": st["device_ms"], "step_ms": ms.get("step_ms")}), file=sys.stderr,
          flush=True)
