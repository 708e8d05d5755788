"""Test helpers: the compiled reference (oracle/_ref, test infrastructure only)
and event-log comparison gates (decision parity required, byte
parity the target)."""
from __future__ import annotations

import ctypes
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libspexref.so"
EMU_SO = ROOT / "build" / "emu" / "libspex_emu.so"
FLOAT_FIELDS = ("r", "weight")

_ref = None


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            return None
        L = ctypes.CDLL(str(REF_SO))
        L.ref_run_log.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p,
                                  ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double)]
        L.ref_run_timed.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int,
                                    ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.ref_last_error.restype = ctypes.c_char_p
        _ref = L
    return _ref


def ref_run_log(cfg: str, seed: int, flags: str | None) -> list[str]:
    L = ref_lib()
    out = ctypes.c_char_p()
    tot = (ctypes.c_double * 24)()
    rc = L.ref_run_log(cfg.encode(), seed, None if flags is None else flags.encode(), ctypes.byref(out), tot)
    if rc != 0:
        raise RuntimeError(f"reference failed rc={rc}: {L.ref_last_error().decode()}")
    return out.value.decode().splitlines()


def strip_floats(line: str) -> dict:
    e = json.loads(line)
    for k in FLOAT_FIELDS:
        e.pop(k, None)
    return e


def compare_logs(ref: list[str], got: list[str]) -> dict:
    """Returns {'decision_ok', 'byte_equal', 'byte_diff_lines', 'first_decision_diff', 'float_max_rel'}."""
    res = {"lines_ref": len(ref), "lines_got": len(got), "byte_equal": ref == got,
           "byte_diff_lines": 0, "first_decision_diff": None, "float_max_rel": 0.0}
    if len(ref) != len(got):
        res["decision_ok"] = False
        res["first_decision_diff"] = min(len(ref), len(got))
        return res
    for i, (a, b) in enumerate(zip(ref, got)):
        if a == b:
            continue
        res["byte_diff_lines"] += 1
        ea, eb = json.loads(a), json.loads(b)
        for k in FLOAT_FIELDS:
            if k in ea and k in eb:
                x, y = float(ea[k]), float(eb[k])
                rel = abs(x - y) / max(abs(x), 1e-300)
                res["float_max_rel"] = max(res["float_max_rel"], rel)
        if strip_floats(a) != strip_floats(b) and res["first_decision_diff"] is None:
            res["first_decision_diff"] = i
    res["decision_ok"] = res["first_decision_diff"] is None
    return res


def sweep_configs():
    """Small configs covering every family x flag set (the reference's own
    integration tests use the same families/flags, test_executor.cpp:217-263)."""
    out = []
    for fam in ("rstar_dfs", "rest_hybrid", "rebase_bfs"):
        for fl in ("", "t1", "t3", "t1,t2", "t1,t3", "t1,t2,t3"):
            for seed, noise in ((1, 0.0), (2, 0.05), (5, 0.05)):
                cfg = {"family": fam, "policy": {"width": 4, "max_depth": 10, "target_answers": 6},
                       "workload": {"noise_sigma": noise}, "run": {"batch_size": 6, "n_queries": 6}}
                out.append((f"{fam}-{fl or 'base'}-s{seed}", json.dumps(cfg), seed, fl))
    return out


def edge_configs():
    """Edge cases of the search (the reference's integration tests exercise
    admission staggering, test_executor.cpp:265-286): queued admission
    (batch_size < n_queries), a single query, width 1, depth 1-2, noise-free and
    noisy rewards, T2 with a tiny producer budget, a large speculation window."""
    base = {"policy": {"width": 4, "max_depth": 8, "target_answers": 6}, "workload": {"noise_sigma": 0.05},
            "run": {"batch_size": 6, "n_queries": 6}}
    cases = []

    def add(name, fam, flags, seed=3, **upd):
        c = json.loads(json.dumps(base))
        c["family"] = fam
        for sect, kv in upd.items():
            c.setdefault(sect, {}).update(kv)
        cases.append((name, json.dumps(c), seed, flags))

    for fam in ("rstar_dfs", "rest_hybrid", "rebase_bfs"):
        add(f"{fam}-queued", fam, "t1,t2,t3", run={"batch_size": 2, "n_queries": 9})
        add(f"{fam}-single", fam, "t1,t3", run={"batch_size": 1, "n_queries": 1})
        add(f"{fam}-width1", fam, "t1,t2,t3", policy={"width": 1})
        add(f"{fam}-depth1", fam, "t1,t2", policy={"max_depth": 1, "target_answers": 2})
        add(f"{fam}-depth2-wide", fam, "t1,t3", policy={"width": 12, "max_depth": 2, "target_answers": 12})
        add(f"{fam}-noisy", fam, "t1,t2,t3", 7, workload={"noise_sigma": 0.4})
        add(f"{fam}-tiny-producers", fam, "t1,t2", run={"max_producers": 2})
        add(f"{fam}-specwin", fam, "t1", run={"spec_k": 32})
        add(f"{fam}-depth-widths", fam, "t1,t2,t3", policy={"depth_widths": [6, 3, 2]})
        add(f"{fam}-kv-latency", fam, "t1,t2,t3", hardware={"kv_bytes_per_token": 131072.0, "reward_latency": 0.5})
        add(f"{fam}-skewed", fam, "t1,t3", 11, workload={"skew": 0.6, "answer_alphabet": 12})
    return cases


def random_configs(n=60, seed=2026):
    """Random configurations across the families, flag sets, widths, depths,
    targets, noise, batch/queue sizes, latency and KV pricing (seeded)."""
    import random
    rng = random.Random(seed)
    fams = ("rstar_dfs", "rest_hybrid", "rebase_bfs")
    flagsets = ("", "t1", "t2", "t3", "t1,t2", "t1,t3", "t2,t3", "t1,t2,t3")
    out = []
    for i in range(n):
        fam = rng.choice(fams)
        nq = rng.randint(1, 12)
        cfg = {"family": fam,
               "policy": {"width": rng.randint(1, 10), "max_depth": rng.randint(1, 14),
                          "target_answers": rng.randint(1, 12), "exploration_c": rng.choice([0.5, 1.0, 2.0]),
                          "balance_temperature": rng.choice([0.5, 1.0, 3.0])},
               "workload": {"noise_sigma": rng.choice([0.0, 0.05, 0.2]), "skew": rng.choice([0.0, 0.3]),
                            "answer_alphabet": rng.randint(2, 12)},
               "hardware": {"kv_bytes_per_token": rng.choice([0.0, 131072.0]),
                            "reward_latency": rng.choice([0.05, 0.1, 0.4])},
               "budget": {"tau": rng.choice([1.0, 2.0, 4.0])},
               "termination": {"alpha": rng.choice([0.25, 0.5, 1.0]), "min_frac": rng.choice([0.4, 0.6])},
               "run": {"batch_size": rng.randint(1, nq), "n_queries": nq, "spec_k": rng.randint(1, 12),
                       "max_producers": rng.choice([4, 16, 64])}}
        out.append((f"rand{i}-{fam}", json.dumps(cfg), rng.randint(1, 10000), rng.choice(flagsets)))
    return out


REF_SPLIT_SO = ROOT / "oracle" / "_ref" / "libspexref_split.so"
_ref_split = None


def ref_split_lib():
    """The split mode's oracle (oracle/ref_split.cpp): the reference's executor,
    one thread per rank, coupled by the T2 budget exchange."""
    global _ref_split
    if _ref_split is None:
        if not REF_SPLIT_SO.exists():
            return None
        L = ctypes.CDLL(str(REF_SPLIT_SO))
        L.ref_split_run_log.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_longlong)]
        L.ref_split_last_error.restype = ctypes.c_char_p
        _ref_split = L
    return _ref_split


def ref_split_log(cfg: str, seed: int, flags: str | None, world: int) -> tuple:
    """(rank logs, rank exchange rounds) of one split job."""
    L = ref_split_lib()
    logs = (ctypes.c_char_p * world)()
    tot = (ctypes.c_double * (24 * world))()
    rounds = (ctypes.c_longlong * world)()
    rc = L.ref_split_run_log(cfg.encode(), seed, None if flags is None else flags.encode(), world, 1, logs, tot,
                             rounds)
    if rc != 0:
        raise RuntimeError(f"split reference failed rc={rc}: {L.ref_split_last_error().decode()}")
    return [logs[r].decode().splitlines() for r in range(world)], list(rounds)


def split_configs():
    """T2 configs of every family for the split mode (the exchange only runs
    with T2): queued admission, several widths / noise levels, 12-40 queries."""
    out = []
    for fam in ("rstar_dfs", "rest_hybrid", "rebase_bfs"):
        for fl, q, bs, seed in (("t1,t2", 12, 12, 1), ("t1,t2,t3", 24, 8, 2), ("t1,t2,t3", 40, 40, 5)):
            cfg = {"family": fam, "policy": {"width": 4, "max_depth": 10, "target_answers": 6},
                   "workload": {"noise_sigma": 0.05}, "run": {"batch_size": bs, "n_queries": q, "max_producers": 24}}
            out.append((f"{fam}-{fl.replace(',', '')}-q{q}-s{seed}", json.dumps(cfg), seed, fl))
    return out
