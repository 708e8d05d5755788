"""GPU: standalone PRM scoring (spex_score_batch) against the
fp32 model oracle (oracle/model_ref.py: the same hash-seeded random-init
weights, RMSNorm / RoPE / GQA attention / SwiGLU in fp32, value head +
sigmoid). Tolerance (stated): |score - oracle| <= 2e-3 — bf16 weights and
activations through the tensor-core prefill against fp32 (the executor's PRM
scores meet the same bound in tests/test_model_gpu.py)."""
import numpy as np
import pytest

import paper_2605_10195_b200 as spex
from oracle import model_ref

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,seed", [("small_prm", 7), ("mid_prm", 3)])
def test_score_batch_matches_fp32_oracle(shape, seed):
    rng = np.random.default_rng(seed)
    V = 512 if shape == "small_prm" else 32000
    lens = [1, 2, 15, 16, 17, 40, 131, 300] + list(rng.integers(1, 200, size=8))
    seqs = [rng.integers(0, V, size=int(n)).tolist() for n in lens]
    got = spex.score_batch(shape, seed, seqs)
    ref = model_ref.Model(shape, seed ^ model_ref.PRM_SEED_XOR, prm=True)
    worst = max(abs(g - ref.prm_score(np.array(s, dtype=np.int64))) for g, s in zip(got, seqs))
    assert worst <= 2e-3, worst
    # order independence: each sequence's score is its own
    again = spex.score_batch(shape, seed, seqs[::-1])
    assert again[::-1] == got


def test_score_batch_errors():
    with pytest.raises(spex.TotsimError):
        spex.score_batch("no_such_prm", 1, [[1, 2, 3]])
    with pytest.raises(spex.TotsimError):
        spex.score_batch("small_prm", 1, [[1, 2], []])
    with pytest.raises(spex.TotsimError):
        spex.score_batch("small_prm", 1, [[1, 512]])
