"""Drop-in proof: the reference's OWN integration
tests (proj/tests/test_executor.cpp, unmodified) linked against the B200 path
through the reference-side binding integration/executor_b200.cpp in place of
the reference's executor.cpp / experiment.cpp (oracle/Makefile target
dropin_test_executor). Every Executor / run_once call in those tests — chain
makespan oracle, replay-clean conservation, byte-identical determinism,
zero-noise T1 tree identity, every family with all flags, admission
staggering, run-once and config errors (test_executor.cpp:125-320) — runs the
sm_100a control kernel."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "dropin_test_executor"


def test_reference_executor_tests_pass_on_b200_path():
    if not BIN.exists():
        pytest.skip("oracle/_ref/dropin_test_executor not built (needs /root/reference at build time)")
    p = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(p.stdout[-2000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stderr[-4000:]
    assert "test cases: 8 | 8 passed | 0 failed" in p.stdout, p.stdout


POLICY_BIN = ROOT / "oracle" / "_ref" / "dropin_test_policy"


def test_reference_policy_and_budget_tests_pass_on_b200_hooks():
    """The reference's own tests/test_policy.cpp and tests/test_budget.cpp
    (unmodified) with ucb_score / ucb_select / rebase_widths /
    roofline_k_total / allocate_budgets routed to the device hooks
    (integration/policy_b200.cpp -> csrc/spex_hooks.cu): the KATs of
    test_policy.cpp:57-280 and test_budget.cpp:106-255, brute-force UCB
    oracles on random stars, and the policy_step shapes per family."""
    if not POLICY_BIN.exists():
        pytest.skip("oracle/_ref/dropin_test_policy not built (needs /root/reference at build time)")
    p = subprocess.run([str(POLICY_BIN)], capture_output=True, text=True, timeout=600)
    print(p.stdout[-2000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    assert "| 0 failed" in p.stdout, p.stdout


def test_hooks_match_reference_on_random_problems():
    """Batched device hooks against the compiled reference's functions on
    random inputs (many problems per launch): tests/hooks_check.py."""
    from paper_2605_10195_b200 import _lib
    from tests import hooks_check, refutil
    if refutil.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    hooks_check.check_hooks(_lib.lib(), refutil.ref_lib())


SIM_BIN = ROOT / "oracle" / "_ref" / "dropin_test_sim"


def test_reference_sim_tests_pass_on_b200_content_and_engine_seams():
    """The reference's own tests/test_sim.cpp (unmodified) with
    RewardOracle::token_len / is_terminal / reward / answer_label and
    DecodeEngine::advance on the device (integration/sim_b200.cpp ->
    csrc/spex_hooks.cu): the oracle's purity, reward levels and noise, token
    length distribution, terminal windows, answer correctness (test_sim.cpp:
    155-332) and the decode engine's batching, staggered joins, limits,
    farewell steps, staged cancels and determinism (:334-460)."""
    if not SIM_BIN.exists():
        pytest.skip("oracle/_ref/dropin_test_sim not built (needs /root/reference at build time)")
    p = subprocess.run([str(SIM_BIN)], capture_output=True, text=True, timeout=900)
    print(p.stdout[-2000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    assert "| 0 failed" in p.stdout, p.stdout


TERM_BIN = ROOT / "oracle" / "_ref" / "dropin_test_termination"


def test_reference_termination_and_speculation_tests_pass_on_b200_hooks():
    """The reference's own tests/test_termination.cpp and
    tests/test_speculation.cpp (unmodified) with AnswerTally::should_terminate,
    dfs_speculative_select and bfs_speculative_allocate on the device
    (integration/speculation_b200.cpp -> the control kernel's
    tally_should_terminate, dfs_plan and rebase_widths): the n >= t gate,
    margins, ties, alpha extremes (test_termination.cpp:80-160), Algorithm 1
    against the clone-and-simulate oracle on 60 random trees, planned-child
    identities, distances (test_speculation.cpp:254-345) and the BFS allocation
    cases (:349-391); the rest of both files runs the reference's own code."""
    if not TERM_BIN.exists():
        pytest.skip("oracle/_ref/dropin_test_termination not built (needs /root/reference at build time)")
    p = subprocess.run([str(TERM_BIN)], capture_output=True, text=True, timeout=900)
    print(p.stdout[-2000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    assert "| 0 failed" in p.stdout, p.stdout


TREE_BIN = ROOT / "oracle" / "_ref" / "dropin_test_tree"


def test_reference_tree_tests_pass_on_b200_hooks():
    """The reference's own tests/test_tree.cpp (unmodified) with
    transition_legal and SearchTree::prune_subtree on the device
    (integration/tree_b200.cpp -> the control kernel's transition_legal and
    tombstone prune): lifecycle legality, prune counts, re-prunes, frontier
    filtering and the snapshot round trips of test_tree.cpp."""
    if not TREE_BIN.exists():
        pytest.skip("oracle/_ref/dropin_test_tree not built (needs /root/reference at build time)")
    p = subprocess.run([str(TREE_BIN)], capture_output=True, text=True, timeout=900)
    print(p.stdout[-2000:], p.stderr[-4000:])
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    assert "| 0 failed" in p.stdout, p.stdout
