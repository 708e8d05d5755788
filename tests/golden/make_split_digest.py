"""Pins the split mode on config 4: SHA-256 of each rank's event log from the
split oracle (oracle/ref_split.cpp — the reference's own executor, one thread
per rank, coupled by the T2 budget exchange), built in this container from
/root/reference. Run: python tests/golden/make_split_digest.py"""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from tests import refutil  # noqa: E402

cfg = (ROOT / "configs" / "c4_rest_w4_q4096.json").read_text()
seed, world = 1, 8
logs, rounds = refutil.ref_split_log(cfg, seed, None, world)
out = {"config": "c4_rest_w4_q4096", "seed": seed, "world": world, "rounds": rounds,
       "lines": [len(x) for x in logs], "sha256": [hashlib.sha256("\n".join(x).encode()).hexdigest() for x in logs]}
(ROOT / "tests" / "golden" / "split_c4_w8_digest.json").write_text(json.dumps(out, indent=1) + "\n")
print(out)
