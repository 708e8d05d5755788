"""oracle/control_ref.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

Pure-Python restatement of the reference's control arithmetic on the hot path
(SURVEY.md §8a), each function citing the reference file:line it restates
(paths relative to /root/reference/proj). Pinned against (1) the reference's own
known-answer tests (tests/test_policy.cpp, test_budget.cpp, test_termination.cpp,
test_sim.cpp — values copied into tests/test_oracle_kats.py) and (2) the
reference compiled from its sources (oracle/_ref/libspexref.so) on random
inputs. Whole-run event logs are pinned directly against oracle/_ref and the
committed golden logs (tests/golden/).

Transcendentals use Python's math module (glibc on this platform), i.e. the
same libm the reference links.
"""
from __future__ import annotations

import math

M64 = 0xFFFFFFFFFFFFFFFF
SALT = dict(tokens=0x746F6B656E730001, terminal=0x7465726D00000002, deep=0x6465657000000003,
            golden=0x676F6C6400000004, noise=0x6E6F697300000005, correct=0x636F727200000006,
            label=0x6C61626C00000007, query=0x7175657200000008)


# ----------------------------------------------------------------- rng.hpp:14-58
def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix(h: int, v: int) -> int:
    return splitmix64(h ^ ((v + 0x9E3779B97F4A7C15 + ((h << 6) & M64) + (h >> 2)) & M64))


def extend_hash(h: int, slot: int) -> int:
    return mix(h, slot + 1)


def uniform01(h: int, salt: int) -> float:
    return float(splitmix64(h ^ salt) >> 11) * 2.0 ** -53


def normal01(h: int, salt: int) -> float:
    u1 = uniform01(h, salt)
    u2 = uniform01(h, salt ^ 0xA5A5A5A5A5A5A5A5)
    if u1 <= 0.0:
        u1 = 2.0 ** -53
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


def lognormal_tokens(h: int, salt: int, mu: float, sigma: float, lo: int, hi: int) -> int:
    z = normal01(h, salt)
    v = math.exp(mu + sigma * z)
    n = int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))  # lround
    return max(lo, min(hi, n))


# ------------------------------------------------------------- policy.cpp:25-118
def ucb_score(value: float, cv: int, pv: int, c: float) -> float:
    if cv <= 0 or pv <= 0:
        raise ValueError("ZeroVisits")
    return value + c * math.sqrt(math.log(float(pv)) / cv)


def ucb_select(children, parent_visits: int, c: float) -> int:
    """children: list of (id, visits, value, pruned) in slot order (policy.cpp:32-51)."""
    live = [ch for ch in children if not ch[3]]
    if not live:
        raise ValueError("NoChildren")
    for ch in live:
        if ch[1] == 0:
            return ch[0]
    best, best_s = None, 0.0
    for cid, v, val, _ in live:
        s = ucb_score(val, v, parent_visits, c)
        if best is None or s > best_s:
            best, best_s = cid, s
    return best


def rebase_widths(rewards, budget: int, temperature: float, sum_preserving: bool = False):
    if not rewards:
        raise ValueError("EmptyRewards")
    if budget < 0 or temperature <= 0.0:
        raise ValueError("InvalidArgument")
    n = len(rewards)
    rmax = max(rewards)
    w = [math.exp((r - rmax) / temperature) for r in rewards]
    total = 0.0
    for x in w:
        total += x
    quota = [budget * x / total for x in w]
    if not sum_preserving:
        widths = [int(math.floor(q + 0.5)) for q in quota]  # round half away from zero (q >= 0)
        if all(x == 0 for x in widths) and budget > 0:
            best = 0
            for i in range(1, n):
                if rewards[i] > rewards[best]:
                    best = i
            widths[best] = 1
        return widths
    widths = [int(math.floor(q)) for q in quota]
    frac = [q - wd for q, wd in zip(quota, widths)]
    leftover = budget - sum(widths)
    if leftover > 0:
        order = sorted(range(n), key=lambda i: -frac[i])  # stable
        k = 0
        while leftover > 0:
            widths[order[k % n]] += 1
            leftover -= 1
            k += 1
    return widths


# ------------------------------------------------------------- budget.cpp:23-100
def roofline_k_total(hw: dict, active: int, avg_kv: float = 0.0, cap: int = 1024) -> int:
    compute_slope = hw["flops_per_token"] / hw["peak_compute"]
    memory_slope = avg_kv / hw["mem_bandwidth"]
    weight_time = hw["weight_bytes"] / hw["mem_bandwidth"]
    if compute_slope <= memory_slope:
        b = cap
    else:
        knee = math.ceil(weight_time / (compute_slope - memory_slope))
        b = int(knee) if knee < cap else cap
    return max(0, b - active)


def query_score(capacity: int, hit_ema: float, kv_bytes: float, weight_bytes: float) -> float:
    return capacity * hit_ema * (weight_bytes + kv_bytes)


def allocate_budgets(states, k_total: int, tau: float, weight_bytes: float):
    """states: list of (capacity, hit_ema, kv_bytes) (budget.cpp:45-96)."""
    n = len(states)
    out = [0] * n
    if n == 0 or k_total <= 0:
        return out
    score = [query_score(c, h, kv, weight_bytes) for c, h, kv in states]
    lo, hi = min(score), max(score)
    norm = [(s - lo) / (hi - lo) for s in score] if hi > lo else [0.0] * n
    w = [math.exp(tau * x) for x in norm]
    total = 0.0
    for x in w:
        total += x
    floor_sum = 0
    for i in range(n):
        f = int(math.floor(k_total * w[i] / total))
        floor_sum += f
        out[i] = min(states[i][0], f)
    leftover = k_total - floor_sum
    if leftover > 0:
        order = sorted(range(n), key=lambda i: -score[i])
        progress = True
        while leftover > 0 and progress:
            progress = False
            for idx in order:
                if leftover == 0:
                    break
                if out[idx] < states[idx][0]:
                    out[idx] += 1
                    leftover -= 1
                    progress = True
    return out


def update_hit_rate(ema: float, hit: bool, alpha: float = 0.2) -> float:
    return (1.0 - alpha) * ema + alpha * (1.0 if hit else 0.0)


# -------------------------------------------------------- termination.cpp:7-48
class AnswerTally:
    def __init__(self):
        self.by = {}
        self.n = 0

    def record(self, label: str, w: float):
        if w < 0:
            raise ValueError("NegativeWeight")
        c, s = self.by.get(label, (0, 0.0))
        self.by[label] = (c + 1, s + w)
        self.n += 1

    def leading_label(self) -> str:
        if not self.by:
            raise ValueError("EmptyTally")
        best = None
        for lab in sorted(self.by):
            if best is None or self.by[lab][1] > self.by[best][1]:
                best = lab
        return best

    def should_terminate(self, min_answers: int, alpha: float) -> bool:
        if self.n < min_answers or not self.by:
            return False
        if len(self.by) < 2:
            return True
        first = second = None
        for lab in sorted(self.by):
            agg = self.by[lab]
            if first is None or agg[1] > first[1]:
                second, first = first, agg
            elif second is None or agg[1] > second[1]:
                second = agg
        margin = first[1] - second[1]
        avg2 = second[1] / second[0] if second[0] > 0 else 0.0
        return margin > alpha * avg2


def min_answers(min_frac: float, target: int) -> int:
    """config.cpp:43-45."""
    return int(math.ceil(min_frac * target))


# ------------------------------------------------------------- sim.cpp:54-289
def unique_kv_tokens(members, parent, tokens) -> int:
    """members: list of (tree_id, node, partial); parent/tokens: dict (tree,node)->."""
    total = 0
    seen = set()
    for tree, node, partial in members:
        total += partial
        cur = parent[(tree, node)]
        while cur is not None:
            if (tree, cur) in seen:
                break
            seen.add((tree, cur))
            total += tokens[(tree, cur)]
            cur = parent[(tree, cur)]
    return total


def step_cost(batch_size: int, unique_tokens: int, hw: dict):
    compute = batch_size * hw["flops_per_token"] / hw["peak_compute"]
    memory = (hw["weight_bytes"] + hw["kv_bytes_per_token"] * float(unique_tokens)) / hw["mem_bandwidth"]
    return compute, memory


def elapsed(steps: int, compute: float, mem_a: float, mem_d: float) -> float:
    if steps <= 0:
        return 0.0
    m = float(steps)
    if mem_d <= 0.0:
        return m * max(compute, mem_a)
    i0 = 0
    if compute > mem_a:
        i0 = min(steps, int(math.floor((compute - mem_a) / mem_d)) + 1)
    tail = float(steps - i0)
    return i0 * compute + tail * mem_a + mem_d * (float(i0) + m - 1.0) * tail / 2.0


# ---------------------------------------------------------- sim.cpp:106-198
WORKLOAD_DEFAULTS = dict(token_mu=4.2485, token_sigma=0.30, token_min=8, token_max=400, shallow_min=3,
                         shallow_p=0.30, shallow_max=9, deep_min=11, deep_p=0.25, deep_max=18, skew=0.0,
                         golden_density=0.55, reward_on=0.8, reward_off=0.3, noise_sigma=0.0,
                         correct_base=0.95, correct_slope=0.07, correct_floor=0.15, answer_alphabet=6,
                         prompt_tokens=32)


def token_len(child_hash: int, wl=WORKLOAD_DEFAULTS) -> int:
    return lognormal_tokens(child_hash, SALT["tokens"], wl["token_mu"], wl["token_sigma"], wl["token_min"],
                            wl["token_max"])


def query_seed(run_seed: int, q: int) -> int:
    return mix(splitmix64(run_seed ^ SALT["query"]), q + 1)


def golden_label(qseed: int, alphabet: int = 6) -> int:
    return splitmix64(qseed ^ SALT["label"]) % alphabet


def reward_of_path(path_hashes, wl=WORKLOAD_DEFAULTS) -> float:
    """path_hashes: hashes of the nodes depth 1..d of the path (sim.cpp:139-152)."""
    golden = all(uniform01(h, SALT["golden"]) < wl["golden_density"] for h in path_hashes)
    r = wl["reward_on"] if golden else wl["reward_off"]
    if wl["noise_sigma"] > 0.0:
        r += wl["noise_sigma"] * normal01(path_hashes[-1], SALT["noise"])
    return min(1.0, max(0.0, r))
