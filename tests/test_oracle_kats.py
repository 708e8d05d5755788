"""CPU: the oracle restatement (oracle/control_ref.py) against the reference's
own known-answer tests (values from /root/reference/proj/tests/*.cpp, cited per
check) and against the reference compiled from its sources (oracle/_ref) on
random inputs."""
import ctypes
import math
import random

import pytest

from oracle import control_ref as cr
from tests import refutil

HW = dict(weight_bytes=14e9, mem_bandwidth=7e11, peak_compute=1e14, flops_per_token=14e9,
          kv_bytes_per_token=0.0, reward_latency=0.1)


def test_ucb_kats():  # test_policy.cpp:57-60
    assert cr.ucb_score(0.5, 1, 1, 1.0) == pytest.approx(0.5, rel=1e-12)
    assert cr.ucb_score(0.4, 2, 8, 1.0) == pytest.approx(1.419666990168809, rel=1e-9)
    assert cr.ucb_score(0.0, 1, 3, 2.0) == pytest.approx(2.0 * math.sqrt(math.log(3.0)), rel=1e-12)
    with pytest.raises(ValueError):
        cr.ucb_score(0.5, 0, 4, 1.0)


def test_rebase_width_kats():  # test_policy.cpp:203-208,234-237
    assert cr.rebase_widths([0.7, 0.7, 0.7], 9, 1.0) == [3, 3, 3]
    assert cr.rebase_widths([0.7, 0.7, 0.7], 9, 0.01) == [3, 3, 3]
    assert cr.rebase_widths([1.0, 0.5, 0.0], 8, 1.0) == [4, 2, 1]
    assert cr.rebase_widths([1.0, 0.5, 0.0], 8, 1.0, sum_preserving=True) == [4, 2, 2]
    assert cr.rebase_widths([0.2, 0.8, 0.4], 1, 1e6) == [0, 1, 0]


def test_roofline_kats():  # test_budget.cpp:106-137
    assert cr.roofline_k_total(HW, 0) == 143
    assert cr.roofline_k_total(HW, 16) == 127
    assert cr.roofline_k_total(HW, 143) == 0
    assert cr.roofline_k_total(HW, 0, 1e8) == 1024
    assert cr.roofline_k_total(HW, 24, 1e8) == 1000
    assert cr.roofline_k_total(HW, 0, 1e8, 64) == 64
    p2 = dict(HW, weight_bytes=2.0 ** 34, mem_bandwidth=2.0 ** 39, flops_per_token=2.0 ** 33, peak_compute=2.0 ** 48)
    assert cr.roofline_k_total(p2, 0, 0.0, 4096) == 1024
    assert cr.roofline_k_total(p2, 1000, 0.0, 4096) == 24


def test_allocation_kats():  # test_budget.cpp:151-182
    assert cr.query_score(4, 0.5, 2e9, 14e9) == 3.2e10
    assert cr.allocate_budgets([(4, 0.5, 0.0)], 6, 2.0, 14e9) == [4]
    assert cr.allocate_budgets([(8, 0.5, 0.0), (8, 0.5, 0.0)], 6, 2.0, 14e9) == [3, 3]
    assert cr.allocate_budgets([(2, 1.0, 0.0), (8, 0.1, 0.0)], 8, math.log(3.0), 14e9) == [2, 2]
    assert cr.allocate_budgets([], 8, 2.0, 14e9) == []
    assert cr.allocate_budgets([(4, 0.5, 0.0)], 0, 2.0, 14e9) == [0]


def test_termination_kats():  # termination.cpp:30-48 semantics, config.cpp:43-45
    t = cr.AnswerTally()
    for lab, w in [("a1", 0.8), ("a1", 0.8), ("a2", 0.3)]:
        t.record(lab, w)
    assert t.leading_label() == "a1"
    assert t.should_terminate(3, 0.5)
    assert not t.should_terminate(4, 0.5)
    solo = cr.AnswerTally()
    solo.record("a3", 0.1)
    assert solo.should_terminate(1, 0.5)
    assert cr.min_answers(0.6, 10) == 6 and cr.min_answers(0.6, 8) == 5


def test_elapsed_matches_step_sum():  # sim.cpp:277-289 against direct summation
    for compute, mem_a, mem_d in [(0.02, 0.01, 0.001), (0.01, 0.02, 0.0005), (0.02, 0.02, 0.0)]:
        for steps in range(0, 40):
            direct = sum(max(compute, mem_a + i * mem_d) for i in range(steps))
            assert cr.elapsed(steps, compute, mem_a, mem_d) == pytest.approx(direct, rel=1e-12, abs=1e-15)


def test_unique_kv_prefix_sharing():  # test_sim.cpp:52-70
    parent = {(0, 0): None, (0, 1): 0, (0, 2): 1, (0, 3): 1, (0, 4): 0, (0, 5): 4}
    tokens = {(0, 0): 32, (0, 1): 100, (0, 2): 60, (0, 3): 60, (0, 4): 100, (0, 5): 60}
    assert cr.unique_kv_tokens([(0, 2, 10), (0, 3, 20)], parent, tokens) == 162
    assert cr.unique_kv_tokens([(0, 2, 10), (0, 5, 20)], parent, tokens) == 262
    assert cr.unique_kv_tokens([(0, 2, 10), (0, 2, 10)], parent, tokens) == 152


@pytest.mark.skipif(refutil.ref_lib() is None, reason="oracle/_ref not built")
def test_restatement_matches_compiled_reference_random():
    L = refutil.ref_lib()
    L.ref_rebase_widths.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.ref_allocate_budgets.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    L.ref_token_len.argtypes = [ctypes.c_uint64]
    L.ref_normal01.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    L.ref_normal01.restype = ctypes.c_double
    L.ref_splitmix64.argtypes = [ctypes.c_uint64]
    L.ref_splitmix64.restype = ctypes.c_uint64
    rng = random.Random(7)
    for _ in range(300):
        n = rng.randint(1, 9)
        rs = [rng.random() for _ in range(n)]
        budget, temp, sp = rng.randint(0, 20), 0.25 * rng.randint(1, 8), rng.random() < 0.5
        out = (ctypes.c_int * n)()
        assert L.ref_rebase_widths((ctypes.c_double * n)(*rs), n, budget, temp, int(sp), out) == 0
        assert list(out) == cr.rebase_widths(rs, budget, temp, sp)
    hw6 = (ctypes.c_double * 6)(14e9, 7e11, 1e14, 14e9, 0.0, 0.1)
    for _ in range(300):
        n = rng.randint(1, 12)
        st = [(rng.randint(0, 8), rng.random(), rng.random() * 1e10) for _ in range(n)]
        k = rng.randint(0, 40)
        out = (ctypes.c_int * n)()
        L.ref_allocate_budgets((ctypes.c_int * n)(*[s[0] for s in st]), (ctypes.c_double * n)(*[s[1] for s in st]),
                               (ctypes.c_double * n)(*[s[2] for s in st]), n, k, 2.0, hw6, out)
        assert list(out) == cr.allocate_budgets(st, k, 2.0, 14e9)
    for i in range(2000):
        h = rng.getrandbits(64)
        assert L.ref_splitmix64(h) == cr.splitmix64(h)
        assert L.ref_token_len(h) == cr.token_len(h)
        assert L.ref_normal01(h, 5) == cr.normal01(h, 5)
