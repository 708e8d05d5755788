"""One search of a config on the control kernel alone (no model, no trace):
the target of the control-kernel ncu source capture."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rebase_w16_q256"
cfg = (ROOT / "configs" / f"{name}.json").read_text()
ex = spex.Executor(cfg, json.loads(cfg)["run"]["seed"], None, trace=False)
t = ex.run()
print(json.dumps({"cfg": name, "queries": t.queries, "device_ms": ex.stats()["device_ms"]}))
ex.close()
