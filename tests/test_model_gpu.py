"""GPU numerics of the policy / PRM forward vs the numpy fp32 restatement
(oracle/model_ref.py). The reference has no model, so this parity is
*unpinned* against it; the oracle recomputes each sampled row
by a full causal forward over its root->node token sequence, independently of
the device's incremental tree-KV decode.

Tolerances (stated, north_star's 1e-3 relative at bf16 against fp32):
logsumexp |d| <= 1e-3 * max(1, |lse|); logit sum |d| <= 1e-3 * sum |z| (a sum
of V fp32 logits); argmax equal unless the top-2 logits are within
2e-3 * max(1, |lse|) (each logit within 1e-3 * max(1, |lse|)); PRM score
|d| <= 1e-3 * |score|.
"""
import json
import random
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_small_model_matches_numpy_oracle():
    import paper_2605_10195_b200 as spex
    from oracle import model_ref
    if not spex.device_ok():
        pytest.fail("no sm_100 device")
    cfg = (ROOT / "configs" / "c1_rebase_w4_q16.json").read_text()
    seed = json.loads(cfg)["run"]["seed"]
    ex = spex.Executor(cfg, seed, None, trace=True)
    ex.set_model("small_policy", "small_prm", weight_seed=7, record_outputs=True)
    ex.run()
    log = ex.log_lines()
    dec = ex.decode_outputs()
    prm = ex.prm_outputs()
    ms = ex.model_stats()
    ex.close()
    assert ms["decode_rows"] == len(dec) > 0
    assert ms["prm_thoughts"] == len(prm) > 0
    tree = model_ref.TreeFromLog(log, prompt_tokens=32)
    pol = model_ref.Model("small_policy", 7, prm=False)
    rm = model_ref.Model("small_prm", 7 ^ model_ref.PRM_SEED_XOR, prm=True)
    rng = random.Random(0)
    worst = {"lse": 0.0, "sum": 0.0, "prm": 0.0}
    for (q, node, pos, amax, lse, lsum) in rng.sample(dec, 60):
        toks = tree.sequence(q, node, pos, pol.V)
        ra, rl, rs, z = pol.logits_stats(toks)
        worst["lse"] = max(worst["lse"], abs(rl - lse))
        worst["sum"] = max(worst["sum"], abs(rs - lsum))
        assert abs(rl - lse) <= 1e-3 * max(1.0, abs(rl)), (q, node, pos, rl, lse)
        assert abs(rs - lsum) <= 1e-3 * float(np.abs(z).sum()), (q, node, pos, rs, lsum)
        if amax != ra:
            assert z[ra] - z[amax] <= 2e-3 * max(1.0, abs(rl)), (q, node, pos, ra, amax)
    for (q, node, score) in rng.sample(prm, 30):
        n = tree.nodes[(q, node)][2]
        toks = tree.sequence(q, node, n - 1, rm.V)
        rs = rm.prm_score(toks)
        worst["prm"] = max(worst["prm"], abs(rs - score))
        assert abs(rs - score) <= 1e-3 * abs(rs), (q, node, rs, score)
    print("worst abs errors", worst)


def test_mid_model_tensor_core_paths_match_numpy_oracle():
    """dh=128 shapes: PRM/prompt rows go through the TMA + mma.sync tile kernel,
    decode rows through the streaming decode kernel."""
    import paper_2605_10195_b200 as spex
    from oracle import model_ref
    cfg = json.dumps({"family": "rebase_bfs", "policy": {"width": 3, "max_depth": 6, "target_answers": 3},
                      "workload": {"noise_sigma": 0.05}, "run": {"batch_size": 3, "n_queries": 3, "flags": ["t1"]}})
    ex = spex.Executor(cfg, 5, None, trace=True)
    ex.set_model("mid_policy", "mid_prm", weight_seed=3, record_outputs=True)
    ex.run()
    log, dec, prm = ex.log_lines(), ex.decode_outputs(), ex.prm_outputs()
    ex.close()
    assert dec and prm
    tree = model_ref.TreeFromLog(log, prompt_tokens=32)
    rm = model_ref.Model("mid_prm", 3 ^ model_ref.PRM_SEED_XOR, prm=True)
    rng = random.Random(1)
    for (q, node, score) in rng.sample(prm, 4):
        n = tree.nodes[(q, node)][2]
        rs = rm.prm_score(tree.sequence(q, node, n - 1, rm.V))
        assert abs(rs - score) <= 1e-3 * abs(rs), (q, node, rs, score)
    pol = model_ref.Model("mid_policy", 3, prm=False)
    for (q, node, pos, amax, lse, lsum) in rng.sample(dec, 2):
        _, rl, rs, _ = pol.logits_stats(tree.sequence(q, node, pos, pol.V))
        assert abs(rl - lse) <= 1e-3 * max(1.0, abs(rl)), (q, node, pos, rl, lse)
