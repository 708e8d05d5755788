"""Regenerates tests/golden/*.jsonl.gz from the reference simulator compiled by
oracle/Makefile (oracle/_ref/libspexref.so). Run here, where /root/reference
exists; the fixtures travel with the repo so GPU tests and smoke() need neither
/root/reference nor oracle/_ref."""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from tests import refutil  # noqa: E402

CASES = [
    ("c1_rebase_w4_q16", (ROOT / "configs" / "c1_rebase_w4_q16.json").read_text(), 1, None),
    ("c1_rebase_w4_q16_baseline", (ROOT / "configs" / "c1_rebase_w4_q16.json").read_text(), 1, ""),
]
for fam in ("rstar_dfs", "rest_hybrid", "rebase_bfs"):
    cfg = {"family": fam, "policy": {"width": 4, "max_depth": 10, "target_answers": 6},
           "workload": {"noise_sigma": 0.05}, "run": {"batch_size": 3, "n_queries": 5}}
    CASES.append((f"small_{fam}_t123", json.dumps(cfg), 11, "t1,t2,t3"))
    CASES.append((f"small_{fam}_base", json.dumps(cfg), 11, ""))

manifest = []
for name, cfg, seed, flags in CASES:
    lines = refutil.ref_run_log(cfg, seed, flags)
    out = ROOT / "tests" / "golden" / f"{name}.jsonl.gz"
    with gzip.open(out, "wt") as f:
        f.write("\n".join(lines) + "\n")
    manifest.append({"name": name, "config": json.loads(cfg), "seed": seed, "flags": flags, "lines": len(lines)})
(ROOT / "tests" / "golden" / "manifest.json").write_text(json.dumps(manifest, indent=1))
print("wrote", len(manifest), "golden logs")
