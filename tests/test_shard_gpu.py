"""Query-sharded model work with the search replicated (SURVEY.md §8e,
`spex_executor_set_shard`): rank r of W runs the policy/PRM forward only for
queries [Q*r/W, Q*(r+1)/W) while its control kernel runs the whole search.

Checked on one GPU by running every rank of W in turn:
  * each rank's event log is byte-identical to the unsharded run (so to the
    reference's single-server log: one virtual clock, global T2 budgets);
  * the shards partition the model work exactly: decode rows, decode steps'
    rows, PRM thoughts/rows and prefill rows sum to the unsharded totals, and
    K1's algorithmic bytes (unique KV tokens are per tree) sum to the total;
  * every recorded decode / PRM output of a rank belongs to its block, and the
    union over ranks equals the unsharded outputs keyed by (q, node, pos):
    lse within 2e-3 * max(1, |lse|), PRM scores within 2e-3, token ids equal
    but for at most 0.5% near-tie flips (batch composition may change the
    GEMM blocking).
"""
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(cfg, seed, flags, rank=None, world=None):
    import paper_2605_10195_b200 as spex
    ex = spex.Executor(cfg, seed, flags, trace=True)
    ex.set_model("small_policy", "small_prm", weight_seed=7, record_outputs=True)
    if world is not None:
        ex.set_shard(rank, world)
    ex.run()
    out = (ex.log_lines(), ex.model_stats(), ex.decode_outputs(), ex.prm_outputs())
    ex.close()
    return out


@pytest.mark.parametrize("name,flags,world", [("c1_rebase_w4_q16", None, 2), ("c1_rebase_w4_q16", "t1,t2,t3", 3),
                                              ("c1_rebase_w4_q16", "t1", 16)])
def test_shards_partition_model_work_with_identical_logs(name, flags, world):
    import paper_2605_10195_b200 as spex
    if not spex.device_ok():
        pytest.fail("no sm_100 device: the B200 path has no fallback")
    cfg = (ROOT / "configs" / f"{name}.json").read_text()
    Q = json.loads(cfg)["run"]["n_queries"]
    seed = json.loads(cfg)["run"]["seed"]
    log, ms, dec, prm = _run(cfg, seed, flags)
    assert ms["decode_rows"] == len(dec) > 0 and ms["prm_thoughts"] == len(prm) > 0
    full_dec = {(q, n, p): (a, l) for (q, n, p, a, l, _s) in dec}
    full_prm = {(q, n): s for (q, n, s) in prm}
    assert len(full_dec) == len(dec) and len(full_prm) == len(prm)
    tot = {k: 0 for k in ("decode_rows", "prm_thoughts", "prm_rows", "prefill_rows")}
    alg = 0.0
    seen_dec, seen_prm = set(), set()
    flips = 0
    for r in range(world):
        lo, hi = Q * r // world, Q * (r + 1) // world
        lg, m, d, p = _run(cfg, seed, flags, r, world)
        assert lg == log, f"rank {r}: event log differs from the unsharded run"
        for k in tot:
            tot[k] += m[k]
        alg += m["attn_alg_bytes"]
        assert m["decode_rows"] == len(d) and m["prm_thoughts"] == len(p)
        for (q, n, pos, a, lse, _s) in d:
            assert lo <= q < hi, (r, q)
            key = (q, n, pos)
            assert key not in seen_dec
            seen_dec.add(key)
            fa, fl = full_dec[key]
            assert abs(fl - lse) <= 2e-3 * max(1.0, abs(fl)), (key, fl, lse)
            flips += a != fa
        for (q, n, s) in p:
            assert lo <= q < hi, (r, q)
            assert (q, n) not in seen_prm
            seen_prm.add((q, n))
            assert abs(full_prm[(q, n)] - s) <= 2e-3, ((q, n), full_prm[(q, n)], s)
    for k in tot:
        assert tot[k] == ms[k], (k, tot[k], ms[k])
    assert seen_dec == set(full_dec) and seen_prm == set(full_prm)
    assert flips <= max(2, len(dec) // 200), flips  # near-tie argmax flips only
    assert abs(alg - ms["attn_alg_bytes"]) <= 1e-9 * ms["attn_alg_bytes"]


def test_set_shard_rejects_bad_rank():
    import paper_2605_10195_b200 as spex
    cfg = (ROOT / "configs" / "c1_rebase_w4_q16.json").read_text()
    ex = spex.Executor(cfg, 1, None)
    with pytest.raises(spex.TotsimError):
        ex.set_shard(2, 2)
    with pytest.raises(spex.TotsimError):
        ex.set_shard(0, 0)
    ex.close()
