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
