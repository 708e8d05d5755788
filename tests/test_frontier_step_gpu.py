"""GPU: stepwise execution on the sm_100a control kernel (spex_frontier_step,
SURVEY.md §8b): the run's state stays on the device between launches; the
concatenated per-call events equal the compiled reference's run_once log byte
for byte."""
from pathlib import Path

import pytest

import paper_2605_10195_b200 as spex
from tests import refutil

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
needs_ref = pytest.mark.skipif(refutil.ref_lib() is None, reason="oracle/_ref not built")


def stepped(cfg, seed, flags, sizes):
    ex = spex.Executor(cfg, seed, flags, trace=True)
    lines, k = [], 0
    while True:
        done, ev = ex.step(sizes[k % len(sizes)])
        lines += ev
        k += 1
        if done:
            break
    full = ex.log_lines()
    ex.close()
    return lines, full, k


@needs_ref
@pytest.mark.parametrize("name,sizes", [("c1_rebase_w4_q16", [1]), ("c1_rebase_w4_q16", [5, 50]),
                                        ("c3_rstar_w4_q512", [1000, 1, 333]), ("c2_rebase_w16_q256", [4000])])
def test_stepped_matches_reference(name, sizes):
    cfg = (ROOT / "configs" / f"{name}.json").read_text()
    ref = refutil.ref_run_log(cfg, 1, None)
    lines, full, calls = stepped(cfg, 1, None, sizes)
    assert lines == ref
    assert full == ref
    assert calls > 1


@needs_ref
@pytest.mark.parametrize("name,cfg,seed,flags", refutil.sweep_configs()[::5])
def test_stepped_sweep(name, cfg, seed, flags):
    lines, _, _ = stepped(cfg, seed, flags, [3, 11])
    assert lines == refutil.ref_run_log(cfg, seed, flags), name


def test_step_refuses_a_model_run():
    cfg = (ROOT / "configs" / "c1_rebase_w4_q16.json").read_text()
    ex = spex.Executor(cfg, 1, None, trace=True)
    ex.set_model("small_policy", "small_prm", 1)
    with pytest.raises(spex.TotsimError):
        ex.step(1)
    ex.close()


@needs_ref
def test_spex_run_streams_the_reference_log():
    cfg = (ROOT / "configs" / "c3_rstar_w4_q512.json").read_text()
    got = []
    t = spex.run(cfg, 1, None, on_event=got.append, chunk=2000)
    ref = refutil.ref_run_log(cfg, 1, None)
    assert got == ref
    assert t.queries == 512
