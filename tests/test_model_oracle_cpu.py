"""Pins the torch restatement of the model oracle (oracle/model_ref_torch.py,
used to check the Llama-3-8B / 1.5B-PRM named shapes on the GPU) to the numpy
restatement (oracle/model_ref.py) on the shapes numpy runs quickly: identical
counter-hash weights bit for bit, and the same logits / PRM scores up to fp32
accumulation order (stated tolerance: logsumexp 1e-4 relative, PRM score 1e-3 relative — one bf16 rounding flip at a quantisation point moves a score ~1e-4)."""
import numpy as np
import pytest
import torch

from oracle import model_ref, model_ref_torch


@pytest.mark.parametrize("shape,tid,scale", [("small_policy", 1, 1.7320508), ("mid_prm", 102, 0.02 * 1.7320508)])
def test_weights_bit_identical(shape, tid, scale):
    n = 100_003
    a = model_ref.init_tensor(n, 7, tid, np.float32(scale))
    b = model_ref_torch.init_tensor(n, 7, tid, float(np.float32(scale)), "cpu").to(torch.float32).numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_hash_constants_match():
    x = torch.tensor([0, 1, 12345, -1, 2 ** 62], dtype=torch.int64)
    got = model_ref_torch._splitmix64(x).numpy().view(np.uint64)
    want = [model_ref.splitmix64(int(v) & ((1 << 64) - 1)) for v in x.tolist()]
    assert [int(g) for g in got] == want


@pytest.mark.parametrize("pol,prm,seed", [("small_policy", "small_prm", 7), ("mid_policy", "mid_prm", 3)])
def test_forward_matches_numpy(pol, prm, seed):
    torch.set_num_threads(4)
    rng = np.random.default_rng(seed)
    P = model_ref.Model(pol, seed, prm=False)
    Pt = model_ref_torch.Model(pol, seed, prm=False)
    toks = rng.integers(0, P.V, 37)
    a, lse, s, _ = P.logits_stats(toks)
    ta, tl, ts, gap = Pt.logits_stats_all(toks, [len(toks) - 1])
    assert abs(tl[0] - lse) <= 1e-4 * max(1.0, abs(lse))
    assert abs(ts[0] - s) <= 1e-3 * np.sqrt(P.V)
    assert ta[0] == a or gap[0] <= 1e-3
    R = model_ref.Model(prm, seed ^ model_ref.PRM_SEED_XOR, prm=True)
    Rt = model_ref_torch.Model(prm, seed ^ model_ref.PRM_SEED_XOR, prm=True)
    toks = rng.integers(0, R.V, 29)
    assert abs(R.prm_score(toks) - Rt.prm_score(toks)) <= 1e-3 * abs(R.prm_score(toks))
