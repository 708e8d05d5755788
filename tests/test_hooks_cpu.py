"""CPU: the policy / budget hooks of the C ABI, evaluated by the test-only
host emulation library (the same control functions, single thread), against
the compiled reference on random problems (tests/hooks_check.py)."""
import pytest

from paper_2605_10195_b200 import _lib
from tests import hooks_check, refutil


def test_emulated_hooks_match_reference():
    if not refutil.EMU_SO.exists():
        pytest.skip("emulation library not built (make -C paper_2605_10195_b200/csrc emu)")
    if refutil.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    hooks_check.check_hooks(_lib.bind(refutil.EMU_SO), refutil.ref_lib())
