"""CPU: the experiment harness (treatment + baseline pairs over repetitions,
aggregation, critical-path savings; experiment.cpp:50-191) over the control
path — the test-only emulation library runs the batched searches — equals the
reference's run_experiment_full metrics (oracle/_ref)."""
import ctypes
import json

import pytest

from paper_2605_10195_b200 import RunTotals, _lib
from paper_2605_10195_b200.experiment import aggregate, compute_critical_path_savings
from tests import refutil

CASES = [
    {"family": "rebase_bfs", "policy": {"width": 4, "max_depth": 8, "target_answers": 6},
     "workload": {"noise_sigma": 0.05}, "run": {"batch_size": 4, "n_queries": 4, "flags": ["t1", "t2", "t3"],
                                                "repetitions": 3, "seed": 5}},
    {"family": "rstar_dfs", "policy": {"width": 4, "max_depth": 8, "target_answers": 6},
     "workload": {"noise_sigma": 0.05}, "run": {"batch_size": 3, "n_queries": 5, "flags": ["t1", "t3"],
                                                "repetitions": 2, "seed": 2}},
    {"family": "rest_hybrid", "policy": {"width": 4, "max_depth": 8, "target_answers": 6},
     "workload": {"noise_sigma": 0.1}, "run": {"batch_size": 4, "n_queries": 4, "repetitions": 2}},
]


def _emu():
    if not refutil.EMU_SO.exists():
        pytest.skip("emulation library not built")
    return _lib.bind(refutil.EMU_SO)


def _batch(L, cfg, seeds, flags):
    arr = (ctypes.c_uint64 * len(seeds))(*seeds)
    tots = (_lib.Totals * len(seeds))()
    ms = ctypes.c_double()
    assert L.spex_run_batch(cfg.encode(), arr, len(seeds), flags, 0, tots, ctypes.byref(ms)) == 0
    return [RunTotals(**t.as_dict()) for t in tots]


def _log(L, cfg, seed, flags):
    t = _lib.Totals()
    out = ctypes.c_void_p()
    assert L.spex_run_once(cfg.encode(), seed, flags, ctypes.byref(t), ctypes.byref(out)) == 0
    try:
        return ctypes.string_at(out.value).decode().splitlines()
    finally:
        L.spex_free(out)


@pytest.mark.parametrize("case", CASES, ids=[c["family"] for c in CASES])
def test_experiment_metrics_match_reference(case):
    R = refutil.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built")
    L = _emu()
    cfg = json.dumps(case)
    R.ref_run_experiment_json.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    out = ctypes.c_char_p()
    assert R.ref_run_experiment_json(cfg.encode(), ctypes.byref(out)) == 0
    ref = json.loads(out.value.decode())
    run = case["run"]
    reps, seed0 = run.get("repetitions", 1), run.get("seed", 1)
    flags_any = bool(run.get("flags"))
    seeds = [seed0 + r for r in range(reps)]
    treat = _batch(L, cfg, seeds, None)
    base = _batch(L, cfg, seeds, b"") if flags_any else treat
    m = aggregate(treat, base, flags_any, reps, _log(L, cfg, seeds[0], None))
    assert list(m.keys()) == list(ref.keys())
    assert m == ref


def test_critical_path_savings_rejects_truncated_logs():
    with pytest.raises(ValueError):
        compute_critical_path_savings(['{"ev":"run_begin"}', '{"ev":"node","q":0}'])
