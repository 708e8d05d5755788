"""Control kernel alone (no model, no trace) per config with its phase cycle
counters (SPEX_PHASES=1, printed to stderr by the library)."""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("SPEX_PHASES", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2605_10195_b200 as spex  # noqa: E402

for n in sys.argv[1:]:
    cfg = (ROOT / "configs" / f"{n}.json").read_text()
    seed = json.loads(cfg)["run"]["seed"]
    ex = spex.Executor(cfg, seed, None, trace=False)
    t0 = time.time()
    tot = ex.run()
    st = ex.stats()
    ex.close()
    print(json.dumps({"cfg": n, "wall_s": round(time.time() - t0, 3), "device_ms": round(st["device_ms"], 2),
                      "iterations": st["iterations"], "epochs": st["epochs"], "rewards": st["reward_events"],
                      "decode_steps": st["decode_steps"], "nodes": st["nodes"]}), flush=True)
