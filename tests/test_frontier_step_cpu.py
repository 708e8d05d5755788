"""CPU: stepwise execution (spex_frontier_step, the fused frontier step of
SURVEY.md §8b) in the test-only emulation library: stepping a run a few
consumer-loop iterations at a time and concatenating each call's events gives
the run_once log byte for byte, whatever the step sizes. The sm_100a kernel is
checked the same way in tests/test_frontier_step_gpu.py."""
import ctypes
import json
from pathlib import Path

import pytest

from paper_2605_10195_b200 import _lib
from tests import refutil

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())


def emu():
    if not refutil.EMU_SO.exists():
        pytest.skip("emulation library not built (make -C paper_2605_10195_b200/csrc emu)")
    return _lib.bind(refutil.EMU_SO)


def stepped(L, cfg, seed, flags, sizes):
    h = ctypes.c_void_p()
    assert L.spex_executor_create(cfg.encode(), seed, None if flags is None else flags.encode(), 0,
                                  ctypes.byref(h)) == 0
    lines, calls, k = [], 0, 0
    try:
        while True:
            done, out, n = ctypes.c_int(), ctypes.c_void_p(), ctypes.c_size_t()
            rc = L.spex_frontier_step(h, sizes[k % len(sizes)], ctypes.byref(done), ctypes.byref(out), ctypes.byref(n))
            assert rc == 0, L.spex_last_error()
            lines += ctypes.string_at(out.value, n.value).decode().splitlines()
            L.spex_free(out)
            calls += 1
            k += 1
            if done.value:
                break
        # the executor counts as run: a further step is refused, the whole log is there
        done = ctypes.c_int()
        assert L.spex_frontier_step(h, 1, ctypes.byref(done), None, None) != 0
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        assert L.spex_executor_log(h, ctypes.byref(p), ctypes.byref(n)) == 0
        full = ctypes.string_at(p.value, n.value).decode().splitlines()
        L.spex_free(p)
        return lines, full, calls
    finally:
        L.spex_executor_destroy(h)


@pytest.mark.parametrize("case", MANIFEST[:6], ids=[c["name"] for c in MANIFEST[:6]])
@pytest.mark.parametrize("sizes", [[1], [7, 1, 30], [0]], ids=["one", "mixed", "all"])
def test_stepped_log_is_the_run_once_log(case, sizes):
    import gzip
    L = emu()
    with gzip.open(GOLDEN / f"{case['name']}.jsonl.gz", "rt") as f:
        golden = f.read().splitlines()
    lines, full, calls = stepped(L, json.dumps(case["config"]), case["seed"], case["flags"], sizes)
    assert lines == golden
    assert full == golden
    if sizes == [0]:
        assert calls == 1
    if sizes == [1]:
        assert calls > 10


def test_spex_run_streams_the_run_once_log():
    """spex_run: the event lines through a callback as the steps produce them."""
    import gzip
    L = emu()
    case = MANIFEST[0]
    with gzip.open(GOLDEN / f"{case['name']}.jsonl.gz", "rt") as f:
        golden = f.read().splitlines()
    got = []
    cb = _lib.TRACE_CB(lambda line, n, user: got.append(line[:n].decode()))
    t = _lib.Totals()
    flags = case["flags"]
    assert L.spex_run(json.dumps(case["config"]).encode(), case["seed"], None if flags is None else flags.encode(), cb,
                      None, 5, ctypes.byref(t)) == 0, L.spex_last_error()
    assert got == golden
    assert t.queries == json.loads(golden[-1])["queries"]
