"""CPU: the content hooks (RewardOracle on the device's draws,
include/spex.h spex_content_*) in the host emulation library against the
compiled reference's own draws (ref_token_len, and the golden logs' token
lengths / rewards through tests/test_emulation_cpu.py)."""
import ctypes
import random

import pytest

from paper_2605_10195_b200 import _lib
from tests import refutil


class Workload(ctypes.Structure):
    _fields_ = [("token_mu", ctypes.c_double), ("token_sigma", ctypes.c_double), ("token_min", ctypes.c_int),
                ("token_max", ctypes.c_int), ("shallow_min", ctypes.c_int), ("shallow_max", ctypes.c_int),
                ("shallow_p", ctypes.c_double), ("deep_min", ctypes.c_int), ("deep_max", ctypes.c_int),
                ("deep_p", ctypes.c_double), ("skew", ctypes.c_double), ("golden_density", ctypes.c_double),
                ("reward_on", ctypes.c_double), ("reward_off", ctypes.c_double), ("noise_sigma", ctypes.c_double),
                ("correct_base", ctypes.c_double), ("correct_slope", ctypes.c_double),
                ("correct_floor", ctypes.c_double), ("answer_alphabet", ctypes.c_int), ("prompt_tokens", ctypes.c_int)]


def default_workload():
    # WorkloadSpec defaults (sim.hpp:82-108)
    return Workload(4.2485, 0.30, 8, 400, 3, 9, 0.30, 11, 18, 0.25, 0.0, 0.55, 0.8, 0.3, 0.0, 0.95, 0.07, 0.15, 6, 32)


def test_token_len_matches_reference():
    if not refutil.EMU_SO.exists() or refutil.ref_lib() is None:
        pytest.skip("emulation library or oracle/_ref not built")
    L = _lib.bind(refutil.EMU_SO)
    R = refutil.ref_lib()
    R.ref_token_len.argtypes = [ctypes.c_uint64]
    rng = random.Random(5)
    hs = [rng.getrandbits(64) for _ in range(5000)]
    out = (ctypes.c_int * len(hs))()
    wl = default_workload()
    assert L.spex_content_token_len((ctypes.c_uint64 * len(hs))(*hs), len(hs), ctypes.byref(wl), out) == 0
    assert list(out) == [R.ref_token_len(h) for h in hs]
