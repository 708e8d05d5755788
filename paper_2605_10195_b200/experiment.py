"""Experiment harness over the device path — the reference's
``run_experiment_full`` / ``run_experiment`` (proj/src/experiment.cpp:50-138)
and ``compute_critical_path_savings`` (experiment.cpp:140-191).

Every repetition r runs the configured flag set and a flagless baseline under
seed ``cfg.seed + r``; the reference loops over repetitions on OpenMP threads
(experiment.cpp:61-78), here each set of repetitions is ONE launch of the
control kernel with one CTA per search (``run_batch``). Aggregation follows the
reference's order and arithmetic exactly (left-fold means, population standard
deviations), so the metrics equal the reference's for the same config.
"""
from __future__ import annotations

import json
import math
from typing import Any

from . import SpexFlags, canonical_config, run_batch, run_once

HIT_DISTANCES = 5  # metrics.hpp:15 kHitDistances


def _mean(xs):
    s = 0.0
    for x in xs:
        s += x
    return 0.0 if not xs else s / float(len(xs))


def _stddev(xs):
    if len(xs) < 2:
        return 0.0
    mu = _mean(xs)
    s = 0.0
    for x in xs:
        s += (x - mu) * (x - mu)
    return math.sqrt(s / float(len(xs)))


def compute_critical_path_savings(log: list) -> int:
    """Tokens speculation saved on the critical path: promoted-and-kept
    generations (their `ready` token counts) of the query that finished last,
    excluding nodes inside pruned subtrees (experiment.cpp:140-191).
    Raises ValueError (IncompleteLog) on a truncated log."""
    ev = [json.loads(x) if isinstance(x, str) else x for x in log]
    if not ev or ev[0].get("ev") != "run_begin" or ev[-1].get("ev") != "run_end":
        raise ValueError("IncompleteLog: log must open with run_begin and close with run_end")
    crit, crit_t, any_done = -1, -1.0, False
    for e in ev:
        if e.get("ev") != "query_done":
            continue
        any_done = True
        if e["t"] > crit_t:
            crit_t, crit = e["t"], e["q"]
    if not any_done:
        raise ValueError("IncompleteLog: log has no finished query")
    children: dict = {}
    promoted: dict = {}
    roots = []
    for e in ev:
        if e.get("q") != crit:
            continue
        kind = e.get("ev")
        if kind == "node":
            children.setdefault(e["parent"], []).append(e["node"])
        elif kind == "promote":
            promoted[e["node"]] = e["ready"]
        elif kind == "prune":
            roots.append(e["node"])
    dead = set()
    for root in roots:
        stack = [root]
        while stack:
            x = stack.pop()
            if x in dead:
                continue
            dead.add(x)
            stack.extend(children.get(x, []))
    return sum(r for n, r in promoted.items() if n not in dead)


def run_experiment_full(cfg: Any, device: int = 0) -> dict:
    """Returns {"metrics": RunMetrics as ordered dict (metrics.cpp:21-38),
    "treatment_log": rep-0 log, "baseline_log": rep-0 baseline log}."""
    c = canonical_config(cfg)
    text = json.dumps(c)
    reps = int(c["run"]["repetitions"])
    seed0 = int(c["run"]["seed"])
    flags = SpexFlags.from_string(",".join(c["run"]["flags"])) if c["run"]["flags"] else SpexFlags()
    seeds = [seed0 + r for r in range(reps)]
    treat, _ = run_batch(text, seeds, flags, device)
    base = run_batch(text, seeds, "", device)[0] if flags.any() else treat
    t0 = run_once(text, seeds[0], flags)
    b0 = run_once(text, seeds[0], "") if flags.any() else t0

    m = aggregate(treat, base, flags.any(), reps, t0.log)
    return {"metrics": m, "treatment_log": t0.log, "baseline_log": b0.log}


def aggregate(treat, base, flags_any: bool, reps: int, treatment_log0) -> dict:
    """RunMetrics from per-repetition totals (experiment.cpp:86-129)."""
    makespans, speedups, throughputs = [], [], []
    gen = com = reu = was = 0
    hits = [0] * (HIT_DISTANCES + 1)
    misses = [0] * (HIT_DISTANCES + 1)
    q_tot = correct = early = 0
    for t, b in zip(treat, base):
        makespans.append(t.makespan)
        speedups.append(b.makespan / t.makespan if flags_any else 1.0)
        throughputs.append(60.0 * t.queries / t.makespan)
        gen += t.generated_tokens
        com += t.committed_tokens
        reu += t.reused_tokens
        was += t.wasted_tokens
        for d in range(1, HIT_DISTANCES + 1):
            hits[d] += t.hits[d]
            misses[d] += t.misses[d]
        q_tot += t.queries
        correct += t.correct_votes
        early += t.early_terminated
    hit_rate = []
    for d in range(1, HIT_DISTANCES + 1):
        n = hits[d] + misses[d]
        hit_rate.append(-1.0 if n == 0 else float(hits[d]) / float(n))
    m = {
        "makespan": _mean(makespans),
        "makespan_stddev": _stddev(makespans),
        "throughput": _mean(throughputs),
        "speedup": _mean(speedups),
        "speedup_stddev": _stddev(speedups),
        "hit_rate_by_distance": hit_rate,
        "generated_tokens": gen,
        "committed_tokens": com,
        "reused_tokens": reu,
        "wasted_tokens": was,
        "critical_path_tokens_saved": compute_critical_path_savings(treatment_log0),
        "vote_accuracy": 0.0 if q_tot == 0 else float(correct) / float(q_tot),
        "early_termination_rate": 0.0 if q_tot == 0 else float(early) / float(q_tot),
        "repetitions": reps,
        "queries": treat[0].queries if treat else 0,
    }
    # RunMetrics::validate (metrics.cpp:12-19)
    if not m["speedup"] > 0.0 or m["makespan"] < 0.0 or gen != com + reu + was:
        raise ValueError(f"ConfigInvalid: metrics invariants broken: {m}")
    return m


def run_experiment(cfg: Any, device: int = 0) -> dict:
    """RunMetrics of run_experiment_full (experiment.cpp:136-138)."""
    return run_experiment_full(cfg, device)["metrics"]
