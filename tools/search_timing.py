"""Host-side phase timing of whole searches (create / set_model / run / stats /
close) with the library's own [spex timing] marks (SPEX_TIMING=1)."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("SPEX_TIMING", "1")
import paper_2605_10195_b200 as spex  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rebase_w16_q256"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = (ROOT / "configs" / f"{name}.json").read_text()
seed = json.loads(cfg)["run"]["seed"]
for r in range(reps):
    t = [time.perf_counter()]
    ex = spex.Executor(cfg, seed, None, trace=False)
    t.append(time.perf_counter())
    ex.set_model("mid_policy", "mid_prm", weight_seed=1)
    t.append(time.perf_counter())
    tot = ex.run()
    t.append(time.perf_counter())
    st, ms = ex.stats(), ex.model_stats()
    t.append(time.perf_counter())
    ex.close()
    t.append(time.perf_counter())
    d = [1000 * (b - a) for a, b in zip(t, t[1:])]
    print(json.dumps({"rep": r, "create_ms": d[0], "set_model_ms": d[1], "run_ms": d[2], "stats_ms": d[3],
                      "close_ms": d[4], "ctl_ms": st["device_ms"], "model_ms": ms["model_ms"],
                      "attn_ms": ms["attn_ms"]}), flush=True)
