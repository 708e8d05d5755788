"""GPU: the decode engine as a handle (spex_engine_*) against
the reference's own DecodeEngine (oracle/_ref, ref_engine_* over reference
SearchTrees) on random operation sequences: add_stream / cancel / drop /
advance with random readiness, budgets and limits over several trees with
shared ancestors. Every returned clock, finished record (id, tokens,
cancelled, time), count, next_ready and done_tokens must be identical —
floating-point values bit for bit."""
import ctypes
import math

import numpy as np
import pytest

from paper_2605_10195_b200 import _lib
from tests import refutil

pytestmark = pytest.mark.gpu


class Finished(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int), ("tokens_done", ctypes.c_int), ("cancelled", ctypes.c_int),
                ("pad", ctypes.c_int), ("time", ctypes.c_double)]


def ref():
    R = refutil.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built")
    R.ref_tree_create.restype = ctypes.c_void_p
    R.ref_tree_create.argtypes = [ctypes.c_int, ctypes.c_uint64]
    R.ref_tree_add.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int]
    R.ref_tree_destroy.argtypes = [ctypes.c_void_p]
    R.ref_engine_create.restype = ctypes.c_void_p
    R.ref_engine_create.argtypes = [ctypes.POINTER(ctypes.c_double)]
    R.ref_engine_destroy.argtypes = [ctypes.c_void_p]
    R.ref_engine_add_stream.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int,
                                        ctypes.c_double]
    R.ref_engine_cancel.argtypes = [ctypes.c_void_p, ctypes.c_int]
    R.ref_engine_drop.argtypes = [ctypes.c_void_p, ctypes.c_int]
    R.ref_engine_advance.restype = ctypes.c_double
    R.ref_engine_advance.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double] + \
        [ctypes.POINTER(ctypes.c_int)] * 3 + [ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_int)]
    for f in ("ref_engine_done_tokens",):
        getattr(R, f).argtypes = [ctypes.c_void_p, ctypes.c_int]
    for f in ("ref_engine_stream_count", "ref_engine_active_count"):
        getattr(R, f).argtypes = [ctypes.c_void_p]
    R.ref_engine_next_ready.restype = ctypes.c_double
    R.ref_engine_next_ready.argtypes = [ctypes.c_void_p]
    return R


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_engine_handle_matches_reference_engine(seed):
    R = ref()
    L = _lib.lib()
    rng = np.random.default_rng(seed)
    prompt = 32
    hw = (14e9, 7e11, 1e14, 14e9, 131072.0 if seed % 2 else 0.0, 0.1)
    hw_c = (ctypes.c_double * 6)(*hw)
    ref_e = R.ref_engine_create(hw_c)
    h = ctypes.c_void_p()
    assert L.spex_engine_create(ctypes.cast(hw_c, ctypes.c_void_p), 0, ctypes.byref(h)) == 0
    trees, parents, tlen = [], [], []
    for t in range(3):
        tr = R.ref_tree_create(prompt, seed * 10 + t)
        par, ln = [-1], [prompt]
        for _ in range(int(rng.integers(8, 24))):
            p = int(rng.integers(0, len(par)))
            n = int(rng.integers(8, 400))
            assert R.ref_tree_add(tr, p, n) == len(par)
            par.append(p)
            ln.append(n)
        trees.append(tr)
        parents.append(par)
        tlen.append(ln)
    now, next_id, live = 0.0, 0, []
    cap = 256
    fin = (Finished * cap)()
    ids, toks, canc = (ctypes.c_int * cap)(), (ctypes.c_int * cap)(), (ctypes.c_int * cap)()
    times = (ctypes.c_double * cap)()
    steps = 0
    try:
        for _ in range(300):
            op = rng.random()
            if op < 0.45 or not live:
                t = int(rng.integers(0, 3))
                node = int(rng.integers(0, len(parents[t])))
                tokens = int(rng.integers(1, 60))
                ready = now + float(rng.choice([0.0, 0.0, rng.random() * 0.3]))
                anc, c = [], parents[t][node]
                while c >= 0:
                    anc.append(c)
                    c = parents[t][c]
                keys = (ctypes.c_uint64 * max(1, len(anc)))(*[(t << 32) | a for a in anc])
                alen = (ctypes.c_int * max(1, len(anc)))(*[tlen[t][a] for a in anc])
                assert R.ref_engine_add_stream(ref_e, next_id, trees[t], node, tokens, ready) == 0
                assert L.spex_engine_add_stream(h, next_id, node, tokens, ready, keys, alen, len(anc)) == 0
                live.append(next_id)
                next_id += 1
            elif op < 0.55:
                sid = int(rng.choice(live))
                started = ctypes.c_int()
                assert L.spex_engine_cancel(h, sid, ctypes.byref(started)) == 0
                assert started.value == R.ref_engine_cancel(ref_e, sid)
            elif op < 0.6:
                sid = int(rng.choice(live))
                R.ref_engine_drop(ref_e, sid)
                assert L.spex_engine_drop(h, sid) == 0
                live.remove(sid)
            else:
                limit = now + float(rng.random() * 0.6)
                n_r = ctypes.c_int()
                r_now = R.ref_engine_advance(ref_e, now, limit, ids, toks, canc, times, cap, ctypes.byref(n_r))
                n_o, reached = ctypes.c_int(), ctypes.c_double()
                assert L.spex_engine_step(h, now, limit, ctypes.cast(fin, ctypes.c_void_p), cap, ctypes.byref(n_o),
                                          ctypes.byref(reached)) == 0, L.spex_last_error()
                assert reached.value == r_now  # bit for bit
                got = [(fin[i].id, fin[i].tokens_done, fin[i].cancelled, fin[i].time) for i in range(n_o.value)]
                exp = [(ids[i], toks[i], canc[i], times[i]) for i in range(n_r.value)]
                assert got == exp
                for i, *_ in got:
                    live.remove(i)
                now = r_now if math.isfinite(r_now) else now
                steps += 1
            assert L.spex_engine_stream_count(h) == R.ref_engine_stream_count(ref_e)
            assert L.spex_engine_active_count(h) == R.ref_engine_active_count(ref_e)
            assert L.spex_engine_next_ready(h) == R.ref_engine_next_ready(ref_e)
            for sid in live[:8]:
                assert L.spex_engine_done_tokens(h, sid) == R.ref_engine_done_tokens(ref_e, sid)
        assert steps > 50
        # errors as the reference's: a non-positive budget is InvalidArgument
        assert L.spex_engine_add_stream(h, 10 ** 6, 0, 0, now, None, None, 0) != 0
    finally:
        L.spex_engine_destroy(h)
        R.ref_engine_destroy(ref_e)
        for tr in trees:
            R.ref_tree_destroy(tr)
