"""CPU: the event-log validator (paper_2605_10195_b200/replay.py, restating
validate_trace, trace.cpp:94-428) agrees with the reference's validator on the
golden logs and on deliberately corrupted ones."""
import ctypes
import gzip
import json
from pathlib import Path

import pytest

from paper_2605_10195_b200.replay import validate_log
from tests import refutil

GOLDEN = Path(__file__).resolve().parent / "golden"
MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())


def _ref_validate(lines):
    R = refutil.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built")
    R.ref_validate_trace.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    out = ctypes.c_char_p()
    rc = R.ref_validate_trace("\n".join(lines).encode(), ctypes.byref(out))
    assert rc == 0, R.ref_last_error()
    return json.loads(out.value.decode())


def _golden(name):
    with gzip.open(GOLDEN / f"{name}.jsonl.gz", "rt") as f:
        return f.read().splitlines()


def _same(lines):
    ref = _ref_validate(lines)
    got = validate_log(lines)
    assert got.ok == ref["ok"], (got.problems, ref["problems"])
    for k in ("generated", "committed", "reused", "wasted", "queries", "makespan"):
        assert getattr(got, k) == ref[k], k
    assert got.problems == ref["problems"]
    return got


@pytest.mark.parametrize("case", MANIFEST, ids=[c["name"] for c in MANIFEST])
def test_golden_logs_validate_like_the_reference(case):
    assert _same(_golden(case["name"])).ok


def _mutations(lines):
    ev = [json.loads(x) for x in lines]
    out = {}

    def with_change(i, key, val):
        e = dict(ev[i])
        e[key] = val
        return lines[:i] + [json.dumps(e, separators=(",", ":"))] + lines[i + 1:]

    first = {}
    for i, e in enumerate(ev):
        first.setdefault(e["ev"], i)
    if "prune" in first:
        out["prune_count"] = with_change(first["prune"], "count", ev[first["prune"]]["count"] + 1)
    if "done" in first:
        out["done_tokens"] = with_change(first["done"], "tokens", ev[first["done"]]["tokens"] + 3)
    if "node" in first:
        out["slot"] = with_change(first["node"], "slot", 7)
    if "reward" in first:
        out["drop_reward"] = lines[:first["reward"]] + lines[first["reward"] + 1:]
    out["no_run_end"] = lines[:-1]
    out["run_end_generated"] = with_change(len(ev) - 1, "generated", ev[-1]["generated"] + 1)
    return out


@pytest.mark.parametrize("name", ["small_rest_hybrid_t123", "small_rstar_dfs_t123", "c1_rebase_w4_q16"])
def test_corrupted_logs_flagged_like_the_reference(name):
    for kind, lines in _mutations(_golden(name)).items():
        got = _same(lines)
        assert not got.ok, kind
