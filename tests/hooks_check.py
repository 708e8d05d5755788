"""Shared check of the policy / budget hooks (include/spex.h) against the
compiled reference (oracle/_ref, test infrastructure): rebase_widths over 400
random problems per launch in both width modes, allocate_budgets over 60 random
query sets. Used with the product library on the GPU (test_dropin_gpu.py) and
with the host emulation library on the CPU (test_hooks_cpu.py)."""
import ctypes
import random


def check_hooks(L, R):
    rng = random.Random(7)
    # rebase_widths: 400 problems in one launch, both width modes
    for mode in (0, 1):
        probs = [[rng.choice([0.0, 0.3, 0.8, 1.0, rng.random()]) for _ in range(rng.randint(1, 40))]
                 for _ in range(400)]
        budgets = [rng.randint(0, 64) for _ in probs]
        temp = rng.choice([0.25, 0.5, 1.0, 3.0])
        flat = [x for p in probs for x in p]
        offs = [0]
        for p in probs:
            offs.append(offs[-1] + len(p))
        D = ctypes.c_double * len(flat)
        I = ctypes.c_int
        widths = (I * len(flat))()
        status = (I * len(probs))()
        assert L.spex_policy_rebase_widths(D(*flat), (I * len(offs))(*offs), (I * len(budgets))(*budgets), len(probs),
                                           temp, mode, widths, status) == 0
        for k, p in enumerate(probs):
            ref = (I * len(p))()
            R.ref_rebase_widths.argtypes = [ctypes.POINTER(ctypes.c_double), I, I, ctypes.c_double, I,
                                            ctypes.POINTER(I)]
            rc = R.ref_rebase_widths((ctypes.c_double * len(p))(*p), len(p), budgets[k], temp, mode, ref)
            assert rc == status[k]
            assert list(ref) == list(widths[offs[k]:offs[k + 1]]), (k, p, budgets[k], temp, mode)
    # allocate_budgets vs the reference
    R.ref_allocate_budgets.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    for _ in range(60):
        n = rng.randint(1, 700)
        cap = [rng.randint(0, 8) for _ in range(n)]
        ema = [rng.choice([0.5, 0.25, rng.random()]) for _ in range(n)]
        kv = [rng.choice([0.0, 1e6 * rng.random()]) for _ in range(n)]
        k_total = rng.randint(-2, 300)
        tau = rng.choice([0.5, 1.0, 2.0, 4.0])
        hw = [14e9, 7e11, 1e14, 14e9, 0.0, 0.1]
        got = (ctypes.c_int * n)()
        assert L.spex_budget_allocate((ctypes.c_int * n)(*cap), (ctypes.c_double * n)(*ema), (ctypes.c_double * n)(*kv),
                                      n, k_total, tau, hw[0], got) == 0
        ref = (ctypes.c_int * n)()
        R.ref_allocate_budgets((ctypes.c_int * n)(*cap), (ctypes.c_double * n)(*ema), (ctypes.c_double * n)(*kv), n,
                               k_total, tau, (ctypes.c_double * 6)(*hw), ref)
        assert list(got) == list(ref), (n, k_total, tau)
    

    # AnswerTally::should_terminate vs the reference: random answer streams over
    # up to 12 labels (label order = the tally's std::map order of "a<idx>")
    R.ref_should_terminate.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                       ctypes.c_int, ctypes.c_double]
    tallies, refs, params = [], [], []
    for _ in range(400):
        n = rng.randint(0, 14)
        k = rng.randint(1, 12)
        lab = [rng.randrange(k) for _ in range(n)]
        w = [rng.choice([0.0, 1.0, 0.5, rng.random()]) for _ in range(n)]
        min_a = rng.randint(0, 10)
        alpha = rng.choice([0.0, 0.5, 1.0, 1e18])
        agg = {}
        for l, x in zip(lab, w):
            c, s_ = agg.get(f"a{l}", (0, 0.0))
            agg[f"a{l}"] = (c + 1, s_ + x)
        order = sorted(agg)  # std::map<std::string> order
        tallies.append(([agg[o][0] for o in order], [agg[o][1] for o in order], n))
        params.append((min_a, alpha))
        refs.append(R.ref_should_terminate((ctypes.c_int * max(1, n))(*lab), (ctypes.c_double * max(1, n))(*w), n,
                                           min_a, alpha))
    for (min_a, alpha) in sorted(set(params)):
        idx = [i for i, p in enumerate(params) if p == (min_a, alpha)]
        cnt = [c for i in idx for c in tallies[i][0]]
        wts = [x for i in idx for x in tallies[i][1]]
        offs = [0]
        for i in idx:
            offs.append(offs[-1] + len(tallies[i][0]))
        ntot = [tallies[i][2] for i in idx]
        out = (ctypes.c_int * len(idx))()
        assert L.spex_termination_should_terminate((ctypes.c_int * max(1, len(cnt)))(*cnt),
                                                   (ctypes.c_double * max(1, len(wts)))(*wts),
                                                   (ctypes.c_int * len(offs))(*offs), (ctypes.c_int * len(ntot))(*ntot),
                                                   len(idx), min_a, alpha, out) == 0
        assert list(out) == [refs[i] for i in idx], (min_a, alpha)
