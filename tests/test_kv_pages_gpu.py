"""GPU: the paged tree-KV store with page reuse, end to end.

A search runs once with a roomy pool and once with a pool just above its live
peak, so the pages of dead thoughts (pruned, REBASE layers expanded, scored
terminals, finished queries) are handed to new thoughts while the forward —
which lags the control kernel — still streams the schedule. Reuse must not
change a decision (same event log) or an output: every decode row's
logsumexp / argmax equals the roomy run's within 1e-5 relative (the decode
kernels stage 16-token pages either way), every PRM score's logit within 5e-3
(the PRM tile kernel stages 64-token chunks across a thought's runs, so a
split thought moves chunk boundaries and with them the bf16 rounding of the
softmax weights; measured up to 1.5e-3), and sampled rows match the fp32
oracle: logsumexp at 1e-3 relative, PRM scores at 5e-3 on the logit. A pool below the
live peak fails with CapacityTreeKV instead of corrupting KV.
"""
import json
import math
import random
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(cfg, seed, policy, prm, wseed, pages):
    import paper_2605_10195_b200 as spex
    if not spex.device_ok():
        pytest.fail("no sm_100 device: the B200 path has no fallback")
    ex = spex.Executor(cfg, seed, None, trace=True)
    ex.set_model(policy, prm, weight_seed=wseed, record_outputs=True)
    ex.set_kv_pages(pages)
    ex.run()
    out = (ex.log_lines(), ex.decode_outputs(), ex.prm_outputs(), ex.kv_stats(), ex.model_stats())
    ex.close()
    return out


def _logit(s):
    return math.log(s / (1.0 - s))


def _same_outputs(a, b, rel=1e-5, abs_prm_logit=5e-3):
    (log_a, dec_a, prm_a), (log_b, dec_b, prm_b) = a, b
    assert log_a == log_b
    da = {(q, n, p): (am, lse) for (q, n, p, am, lse, _) in dec_a}
    db = {(q, n, p): (am, lse) for (q, n, p, am, lse, _) in dec_b}
    assert da.keys() == db.keys()
    flips = 0
    for k, (am, lse) in da.items():
        am2, lse2 = db[k]
        assert abs(lse - lse2) <= rel * max(1.0, abs(lse)), (k, lse, lse2)
        flips += am != am2
    assert flips <= len(da) // 1000, flips  # only exact logit ties may flip
    pa = {(q, n): s for (q, n, s) in prm_a}
    pb = {(q, n): s for (q, n, s) in prm_b}
    assert pa.keys() == pb.keys()
    for k, s in pa.items():
        assert abs(_logit(s) - _logit(pb[k])) <= abs_prm_logit, (k, s, pb[k])


@pytest.mark.parametrize("cfgname,policy,prm,wseed", [
    ("c1_rebase_w4_q16", "small_policy", "small_prm", 7),
    ("mid_rebase", "mid_policy", "mid_prm", 3),
    ("mid_rest", "mid_policy", "mid_prm", 3),
])
def test_page_reuse_keeps_outputs(cfgname, policy, prm, wseed):
    from oracle import model_ref
    if cfgname == "mid_rebase":
        cfg = json.dumps({"family": "rebase_bfs", "policy": {"width": 4, "max_depth": 8, "target_answers": 6},
                          "workload": {"noise_sigma": 0.05},
                          "run": {"batch_size": 12, "n_queries": 12, "flags": ["t1", "t2", "t3"], "seed": 3}})
    elif cfgname == "mid_rest":
        cfg = json.dumps({"family": "rest_hybrid", "policy": {"width": 3, "max_depth": 8, "target_answers": 4},
                          "workload": {"noise_sigma": 0.05},
                          "run": {"batch_size": 8, "n_queries": 8, "flags": ["t1", "t3"], "seed": 4}})
    else:
        cfg = (ROOT / "configs" / f"{cfgname}.json").read_text()
    seed = json.loads(cfg)["run"].get("seed", 1)
    log, dec, prm_out, kv, ms = _run(cfg, seed, policy, prm, wseed, 0)  # default pool: free HBM
    assert ms["streamed"] == 1
    assert kv["live_pages_end"] == kv["root_pages"], kv
    assert kv["allocated_pages"] < kv["pages"] and kv["fresh_pages"] == kv["allocated_pages"], kv  # no reuse
    tight = kv["peak_pages"] + 25
    log2, dec2, prm2, kv2, ms2 = _run(cfg, seed, policy, prm, wseed, tight)
    assert ms2["streamed"] == 1
    assert kv2["fresh_pages"] <= tight < kv2["allocated_pages"], kv2  # pages were reused
    _same_outputs((log, dec, prm_out), (log2, dec2, prm2))
    # and the reused-page run against the fp32 oracle on sampled rows
    tree = model_ref.TreeFromLog(log2, prompt_tokens=32)
    pol = model_ref.Model(policy, wseed, prm=False)
    rm = model_ref.Model(prm, wseed ^ model_ref.PRM_SEED_XOR, prm=True)
    rng = random.Random(11)
    for (q, node, pos, amax, lse, lsum) in rng.sample(dec2, 6):
        _, rl, _, _ = pol.logits_stats(tree.sequence(q, node, pos, pol.V))
        assert abs(rl - lse) <= 1e-3 * max(1.0, abs(rl)), (q, node, pos, rl, lse)
    for (q, node, score) in rng.sample(prm2, 6):
        n = tree.nodes[(q, node)][2]
        rs = rm.prm_score(tree.sequence(q, node, n - 1, rm.V))
        assert abs(_logit(rs) - _logit(score)) <= 5e-3, (q, node, rs, score)


def test_pool_below_live_peak_fails_loudly():
    import paper_2605_10195_b200 as spex
    cfg = (ROOT / "configs" / "c1_rebase_w4_q16.json").read_text()
    seed = json.loads(cfg)["run"]["seed"]
    _, _, _, kv, _ = _run(cfg, seed, "small_policy", "small_prm", 7, 0)
    ex = spex.Executor(cfg, seed, None, trace=False)
    ex.set_model("small_policy", "small_prm", weight_seed=7)
    ex.set_kv_pages((kv["peak_pages"] + kv["root_pages"]) // 2)
    with pytest.raises(spex.TotsimError) as e:
        ex.run()
    ex.close()
    assert "tree KV pool exhausted" in str(e.value)
