"""GPU: model mode — rewards are the PRM's scores (RewardOracle::reward,
sim.cpp:146-152, realised by the PRM forward, K4) instead of the content
oracle's hash draws.

The control kernel waits on device for each scored thought's PRM batch before
handling its reward event, so the search is steered by the model:
  * every reward event's r is exactly the PRM score of that thought (the
    float the value head wrote, as a double);
  * the log is a valid trace (the lifecycle / prune / conservation validator
    restating the reference's validate_trace, trace.cpp:94-428);
  * two runs give the same log (the forward is deterministic);
  * sampled scores match the fp32 oracle at 1e-3 relative;
  * per-query device wall-clock latencies are reported for SPEX and for the
    barrier-synchronous baseline of the same search.
"""
import json
import random
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(cfg, seed, flags, policy, prm, wseed):
    import paper_2605_10195_b200 as spex
    if not spex.device_ok():
        pytest.fail("no sm_100 device: the B200 path has no fallback")
    ex = spex.Executor(cfg, seed, flags, trace=True)
    ex.set_model(policy, prm, weight_seed=wseed, record_outputs=True)
    ex.set_reward_source("prm")
    tot = ex.run()
    out = (ex.log_lines(), ex.prm_outputs(), ex.query_wall_ms(), ex.model_stats(), tot)
    ex.close()
    return out


@pytest.mark.parametrize("cfgname,policy,prm,wseed", [
    ("c1_rebase_w4_q16", "small_policy", "small_prm", 7),
    ("rstar_small", "small_policy", "small_prm", 5),
    ("rest_mid", "mid_policy", "mid_prm", 3),
])
def test_prm_rewards_steer_the_search(cfgname, policy, prm, wseed):
    from oracle import model_ref
    from paper_2605_10195_b200 import replay
    if cfgname == "rstar_small":
        cfg = json.dumps({"family": "rstar_dfs", "policy": {"width": 3, "max_depth": 8, "target_answers": 4},
                          "run": {"batch_size": 6, "n_queries": 6, "flags": ["t1", "t3"], "seed": 2}})
    elif cfgname == "rest_mid":
        cfg = json.dumps({"family": "rest_hybrid", "policy": {"width": 3, "max_depth": 8, "target_answers": 4},
                          "run": {"batch_size": 8, "n_queries": 8, "flags": ["t1", "t2", "t3"], "seed": 4}})
    else:
        cfg = (ROOT / "configs" / f"{cfgname}.json").read_text()
    seed = json.loads(cfg)["run"].get("seed", 1)
    log, scores, (wall, wait_ms), ms, tot = _run(cfg, seed, None, policy, prm, wseed)
    assert tot.queries == json.loads(cfg)["run"]["n_queries"]
    by_node = {(q, n): s for (q, n, s) in scores}
    rewards = [json.loads(l) for l in log if '"ev":"reward"' in l]
    assert rewards
    for e in rewards:
        s = by_node[(e["q"], e["node"])]
        assert e["r"] == min(1.0, max(0.0, float(s))), (e, s)
    rep = replay.validate_log(log)
    assert rep.ok, rep.problems[:5]
    # deterministic forward: the same search again
    log2, _, _, _, _ = _run(cfg, seed, None, policy, prm, wseed)
    assert log2 == log
    # scores vs the fp32 oracle
    tree = model_ref.TreeFromLog(log, prompt_tokens=32)
    rm = model_ref.Model(prm, wseed ^ model_ref.PRM_SEED_XOR, prm=True)
    for (q, node, score) in random.Random(3).sample(scores, min(6, len(scores))):
        n = tree.nodes[(q, node)][2]
        ref = rm.prm_score(tree.sequence(q, node, n - 1, rm.V))
        assert abs(ref - score) <= 1e-3 * abs(ref), (q, node, ref, score)
    assert all(0.0 < w <= ms["step_ms"] + 1.0 for w in wall), (wall, ms["step_ms"])
    assert wait_ms >= 0.0


def test_model_mode_spex_vs_barrier_sync_latency():
    """The metric's second half on hardware: per-query wall-clock latency of the
    same model-mode search with SPEX (t1) and barrier-synchronous (no flags)."""
    import statistics
    cfg = json.dumps({"family": "rebase_bfs", "policy": {"width": 4, "max_depth": 8, "target_answers": 4},
                      "run": {"batch_size": 16, "n_queries": 16, "flags": ["t1"], "seed": 1}})
    res = {}
    for name, flags in (("spex", None), ("barrier_sync", "")):
        log, _, (wall, wait_ms), ms, tot = _run(cfg, 1, flags, "mid_policy", "mid_prm", 1)
        assert tot.queries == 16 and min(wall) > 0
        res[name] = {"p50_ms": statistics.median(wall), "step_ms": ms["step_ms"], "reward_wait_ms": wait_ms}
    print(res)
    assert res["spex"]["p50_ms"] > 0 and res["barrier_sync"]["p50_ms"] > 0
