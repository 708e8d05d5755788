"""CPU: the device control code, compiled for the host in the TEST-ONLY
emulation library (build/emu/libspex_emu.so, single thread), against the
committed reference golden logs. This checks the control logic on a CPU-only
box; the product path is the sm_100a kernel (tests/test_parity_gpu.py)."""
import ctypes
import gzip
import json
from pathlib import Path

import pytest

from paper_2605_10195_b200 import _lib
from tests import refutil

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def emu():
    if not refutil.EMU_SO.exists():
        pytest.skip("emulation library not built (make -C paper_2605_10195_b200/csrc emu)")
    return _lib.bind(refutil.EMU_SO)


def emu_run(L, cfg, seed, flags):
    t = _lib.Totals()
    out = ctypes.c_void_p()
    rc = L.spex_run_once(cfg.encode(), seed, None if flags is None else flags.encode(), ctypes.byref(t),
                         ctypes.byref(out))
    assert rc == 0, L.spex_last_error()
    try:
        return ctypes.string_at(out.value).decode().splitlines(), t
    finally:
        L.spex_free(out)


MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())


@pytest.mark.parametrize("case", MANIFEST, ids=[c["name"] for c in MANIFEST])
def test_emulation_matches_golden(case):
    L = emu()
    with gzip.open(GOLDEN / f"{case['name']}.jsonl.gz", "rt") as f:
        golden = f.read().splitlines()
    got, t = emu_run(L, json.dumps(case["config"]), case["seed"], case["flags"])
    res = refutil.compare_logs(golden, got)
    assert res["decision_ok"], res
    assert res["byte_equal"], res  # byte parity: glibc's exp/log/cos restated bit for bit (ctl_glibc.h)
    assert t.generated_tokens == t.committed_tokens + t.reused_tokens + t.wasted_tokens


@pytest.mark.skipif(refutil.ref_lib() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("name,cfg,seed,flags", refutil.sweep_configs()[::3])
def test_emulation_sweep_vs_reference(name, cfg, seed, flags):
    L = emu()
    got, _ = emu_run(L, cfg, seed, flags)
    res = refutil.compare_logs(refutil.ref_run_log(cfg, seed, flags), got)
    assert res["decision_ok"] and res["byte_equal"], (name, res)


@pytest.mark.skipif(refutil.ref_lib() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("name,cfg,seed,flags", refutil.edge_configs())
def test_emulation_edge_configs_vs_reference(name, cfg, seed, flags):
    L = emu()
    got, t = emu_run(L, cfg, seed, flags)
    res = refutil.compare_logs(refutil.ref_run_log(cfg, seed, flags), got)
    assert res["decision_ok"] and res["byte_equal"], (name, res)
    assert t.generated_tokens == t.committed_tokens + t.reused_tokens + t.wasted_tokens


def test_emulation_run_batch_equals_single_runs():
    """spex_run_batch (one launch, one search per CTA on the device; sequential
    in the emulation) returns the same totals as separate runs."""
    L = emu()
    cfg = json.dumps({"family": "rest_hybrid", "policy": {"width": 4, "max_depth": 8, "target_answers": 6},
                      "workload": {"noise_sigma": 0.05}, "run": {"batch_size": 5, "n_queries": 5,
                                                                 "flags": ["t1", "t2", "t3"]}})
    seeds = [3, 4, 9]
    arr = (ctypes.c_uint64 * 3)(*seeds)
    tots = (_lib.Totals * 3)()
    ms = ctypes.c_double()
    assert L.spex_run_batch(cfg.encode(), arr, 3, None, 0, tots, ctypes.byref(ms)) == 0
    for k, sd in enumerate(seeds):
        _, t = emu_run(L, cfg, sd, None)
        assert tots[k].as_dict() == t.as_dict()


@pytest.mark.skipif(refutil.ref_lib() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("name,cfg,seed,flags", refutil.random_configs(200, seed=7))
def test_emulation_random_configs_vs_reference(name, cfg, seed, flags):
    L = emu()
    got, _ = emu_run(L, cfg, seed, flags)
    res = refutil.compare_logs(refutil.ref_run_log(cfg, seed, flags), got)
    assert res["decision_ok"] and res["byte_equal"], (name, res)
