"""CPU: the paged tree-KV store's bookkeeping (ctl_core.h kv_release /
kv_unpin, ctl_run.h commit allocation) in the test-only host emulation of the
control code, over the golden configs and the family x flag sweep.

The store must never change a decision (the event log stays the reference's),
and its page accounting must close: at the end of a run every thought page is
back in the free ring exactly once (checked inside the emulation, which fails
the run otherwise), the live pages are the static root prompts, and a pool
smaller than the run's page total but at least its live peak is enough (pages
of dead thoughts are reused). A pool below the live peak fails loudly with
CapacityTreeKV (status 107 + ... see ctl_state.h ERR_CAP_KV)."""
import ctypes
import gzip
import json
from pathlib import Path

import pytest

from paper_2605_10195_b200 import _lib
from tests import refutil

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())
ERR_CAP_KV = 107


def emu():
    if not refutil.EMU_SO.exists():
        pytest.skip("emulation library not built (make -C paper_2605_10195_b200/csrc emu)")
    return _lib.bind(refutil.EMU_SO)


def run_paged(L, cfg: str, seed: int, flags, pages: int):
    h = ctypes.c_void_p()
    rc = L.spex_executor_create(cfg.encode(), seed, None if flags is None else flags.encode(), 0, ctypes.byref(h))
    assert rc == 0, L.spex_last_error()
    try:
        assert L.spex_executor_set_kv_pages(h, pages) == 0
        t = _lib.Totals()
        rc = L.spex_executor_run(h, 1, ctypes.byref(t))
        if rc != 0:
            return rc, L.spex_last_error().decode(), None, None
        out = ctypes.c_void_p()
        n = ctypes.c_size_t()
        assert L.spex_executor_log(h, ctypes.byref(out), ctypes.byref(n)) == 0
        log = ctypes.string_at(out.value, n.value).decode().splitlines()
        L.spex_free(out)
        st = _lib.KvStats()
        assert L.spex_executor_kv_stats(h, ctypes.byref(st)) == 0
        return 0, "", log, st.as_dict()
    finally:
        L.spex_executor_destroy(h)


def check_closed(kv):
    assert kv["live_pages_end"] == kv["root_pages"], kv
    assert kv["freed_pages"] == kv["allocated_pages"] - kv["root_pages"], kv
    assert kv["root_pages"] <= kv["peak_pages"] <= kv["fresh_pages"] <= kv["pages"], kv


@pytest.mark.parametrize("case", MANIFEST, ids=[c["name"] for c in MANIFEST])
def test_paged_store_keeps_decisions_and_reuses_pages(case):
    L = emu()
    with gzip.open(GOLDEN / f"{case['name']}.jsonl.gz", "rt") as f:
        golden = f.read().splitlines()
    cfg = json.dumps(case["config"])
    rc, err, log, kv = run_paged(L, cfg, case["seed"], case["flags"], 1 << 22)
    assert rc == 0, err
    assert refutil.compare_logs(golden, log)["decision_ok"]
    check_closed(kv)
    assert kv["fresh_pages"] == kv["allocated_pages"]  # a roomy pool never reuses
    # a pool of the live peak (plus one thought) forces reuse and still suffices
    tight = kv["peak_pages"] + 25
    rc, err, log2, kv2 = run_paged(L, cfg, case["seed"], case["flags"], tight)
    assert rc == 0, err
    assert log2 == log
    check_closed(kv2)
    if kv["allocated_pages"] > tight:
        assert kv2["fresh_pages"] <= tight < kv2["allocated_pages"]
    # below the live peak the run fails loudly
    if kv["peak_pages"] - kv["root_pages"] > 50:
        rc, err, _, _ = run_paged(L, cfg, case["seed"], case["flags"], kv["peak_pages"] // 2 + kv["root_pages"] // 2)
        assert rc == ERR_CAP_KV, (rc, err)
        assert "tree KV pool exhausted" in err


@pytest.mark.parametrize("name,cfg,seed,flags", refutil.sweep_configs()[1::4])
def test_paged_store_sweep(name, cfg, seed, flags):
    L = emu()
    rc, err, log, kv = run_paged(L, cfg, seed, flags, 1 << 22)
    assert rc == 0, (name, err)
    check_closed(kv)
    rc, err, log2, kv2 = run_paged(L, cfg, seed, flags, kv["peak_pages"] + 25)
    assert rc == 0, (name, err)
    assert log2 == log, name
    check_closed(kv2)
