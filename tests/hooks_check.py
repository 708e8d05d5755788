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

    # dfs_speculative_select vs the reference on random trees (committed scored
    # nodes, in-flight and speculative work, pruned branches, terminal answers)
    check_dfs_plan(L, R, rng)
    check_tree_hooks(L, R, rng)


def random_tree(rng, n):
    parent, status, bits, reward, visits, value = [-1], [3], [2], [0.0], [1], [0.0]
    for i in range(1, n):
        p = rng.randrange(i)
        while status[p] in (6, 7):  # no children under pruned nodes or answers
            p = parent[p] if parent[p] >= 0 else 0
            if p == 0:
                break
        r = rng.random()
        kind = rng.choices(["commit", "expanding", "awaiting", "spec", "specdone", "pruned", "answer", "pending"],
                           [10, 1, 1, 1, 1, 1, 1, 1])[0]
        st = {"commit": 3, "expanding": 1, "awaiting": 2, "spec": 4, "specdone": 5, "pruned": 6, "answer": 7,
              "pending": 0}[kind]
        gen = kind in ("commit", "awaiting", "specdone", "answer")
        has_r = kind in ("commit", "specdone", "answer")
        term = kind == "answer" or (kind == "specdone" and rng.random() < 0.2)
        parent.append(p)
        status.append(st)
        bits.append((1 if term else 0) | (2 if gen else 0) | (4 if has_r else 0))
        reward.append(r if has_r else 0.0)
        visits.append(rng.randint(1, 4) if kind in ("commit", "answer") else 0)
        value.append(r if kind in ("commit", "answer") else 0.0)
    for i in range(n - 1, 0, -1):  # ancestors carry their children's traffic
        visits[parent[i]] = max(visits[parent[i]], sum(visits[j] for j in range(n) if parent[j] == i) + visits[i])
    return parent, status, bits, reward, visits, value


def check_dfs_plan(L, R, rng):
    I32, U8, F64, U32 = ctypes.c_int32, ctypes.c_uint8, ctypes.c_double, ctypes.c_uint32
    R.ref_dfs_plan.argtypes = [ctypes.POINTER(I32), ctypes.POINTER(U8), ctypes.POINTER(U8), ctypes.POINTER(F64),
                               ctypes.POINTER(I32), ctypes.POINTER(F64), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                               ctypes.c_int, ctypes.POINTER(I32), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(U32), ctypes.POINTER(I32), ctypes.POINTER(ctypes.c_int)]
    fn = L.spex_speculation_dfs_plan
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(I32), ctypes.POINTER(U8), ctypes.POINTER(U8), ctypes.POINTER(F64),
                   ctypes.POINTER(I32), ctypes.POINTER(F64), ctypes.POINTER(I32), ctypes.c_int, ctypes.c_int,
                   ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.POINTER(I32), ctypes.c_int, ctypes.c_int,
                   ctypes.c_int, ctypes.POINTER(U32), ctypes.POINTER(I32), ctypes.POINTER(ctypes.c_int)]
    planned = 0
    for trial in range(300):
        n = rng.randint(1, 40)
        parent, status, bits, reward, visits, value = random_tree(rng, n)
        depth = [0] * n
        for i in range(1, n):
            depth[i] = depth[parent[i]] + 1
        family = rng.choice([0, 0, 1, 2])
        c = rng.choice([0.5, 1.0, 1.414])
        width = rng.randint(1, 4)
        dw = [rng.randint(1, 5) for _ in range(rng.randint(0, 3))]
        target = rng.randint(1, 12)
        k = rng.randint(0, 8)
        args = ((I32 * n)(*parent), (U8 * n)(*status), (U8 * n)(*bits), (F64 * n)(*reward), (I32 * n)(*visits),
                (F64 * n)(*value))
        dwa = (I32 * max(1, len(dw)))(*dw)
        rn, rd, rc_n = (U32 * 64)(), (I32 * 64)(), ctypes.c_int()
        rrc = R.ref_dfs_plan(*args, n, family, c, width, dwa, len(dw), target, k, rn, rd, ctypes.byref(rc_n))
        gn, gd, g_n = (U32 * 64)(), (I32 * 64)(), ctypes.c_int()
        terminal_answers = sum(1 for s_ in status if s_ == 7)
        grc = fn(*args, (I32 * n)(*depth), n, terminal_answers, family, c, width, dwa, len(dw), target, k, gn, gd,
                 ctypes.byref(g_n))
        assert (rrc != 0) == (grc != 0), (trial, rrc, grc)
        if rrc:
            continue
        got = [(gn[i], gd[i]) for i in range(g_n.value)]
        exp = [(rn[i], rd[i]) for i in range(rc_n.value)]
        assert got == exp, (trial, family, k, got, exp)
        planned += len(exp)
    assert planned > 100


def check_tree_hooks(L, R, rng):
    """transition_legal on all 64 status pairs; prune_subtree on random trees."""
    U8, I32 = ctypes.c_uint8, ctypes.c_int32
    frm = [a for a in range(8) for _ in range(8)]
    to = [b for _ in range(8) for b in range(8)]
    out = (U8 * 64)()
    assert L.spex_tree_transition_legal((U8 * 64)(*frm), (U8 * 64)(*to), 64, out) == 0
    assert list(out) == [R.ref_transition_legal(a, b) for a, b in zip(frm, to)]
    R.ref_prune_subtree.argtypes = [ctypes.POINTER(I32), ctypes.POINTER(U8), ctypes.c_int, ctypes.c_uint32,
                                    ctypes.POINTER(ctypes.c_int)]
    fn = L.spex_tree_prune_subtree
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(I32), ctypes.POINTER(U8), ctypes.c_int, ctypes.c_uint32, ctypes.POINTER(ctypes.c_int)]
    for _ in range(200):
        n = rng.randint(1, 60)
        parent = [-1] + [rng.randrange(i) for i in range(1, n)]
        status = [rng.randrange(8) for _ in range(n)]
        node = rng.randrange(n + 2)  # sometimes outside the tree: UnknownNode
        a, b = (U8 * n)(*status), (U8 * n)(*status)
        pa, pb = ctypes.c_int(), ctypes.c_int()
        ra = R.ref_prune_subtree((I32 * n)(*parent), a, n, node, ctypes.byref(pa))
        rb = fn((I32 * n)(*parent), b, n, node, ctypes.byref(pb))
        assert ra == rb, (ra, rb)
        assert list(a) == list(b) and pa.value == pb.value
