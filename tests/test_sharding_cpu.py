"""CPU, world_size 2 over gloo: the multi-GPU path's host logic — disjoint
per-rank query sets (shard_seed) and the max/sum report reduction — with each
rank running its shard through the test-only emulation of the control code."""
import ctypes
import json
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import refutil

CFG = json.dumps({"family": "rest_hybrid", "policy": {"width": 3, "max_depth": 8, "target_answers": 4},
                  "workload": {"noise_sigma": 0.05}, "run": {"batch_size": 4, "n_queries": 4}})


def _run_shard(seed):
    from paper_2605_10195_b200 import _lib
    L = _lib.bind(refutil.EMU_SO)
    t = _lib.Totals()
    out = ctypes.c_void_p()
    assert L.spex_run_once(CFG.encode(), seed, b"t1,t2,t3", ctypes.byref(t), ctypes.byref(out)) == 0
    L.spex_free(out)
    return t.queries, t.generated_tokens


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_10195_b200.shard import reduce_report, shard_seed
    queries, gen = _run_shard(shard_seed(100, rank))
    secs = 1.0 + rank
    mx, total = reduce_report(secs, float(queries), group=dist.group.WORLD)
    q.put((rank, queries, gen, mx, total))
    dist.destroy_process_group()


@pytest.mark.skipif(not refutil.EMU_SO.exists(), reason="emulation library not built")
def test_two_rank_sharding_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (_, q0, g0, mx0, tot0), (_, q1, g1, mx1, tot1) = res
    assert q0 == q1 == 4
    assert g0 != g1  # disjoint query sets (different seeds)
    assert mx0 == mx1 == 2.0 and tot0 == tot1 == 8.0
    assert (q0, g0) == _run_shard(100) and (q1, g1) == _run_shard(101)


def _coupled_log(seed, rank, world):
    """One search on the emulation with this rank's query block set; returns
    (serialised event log, totals.queries)."""
    from paper_2605_10195_b200 import _lib
    L = _lib.bind(refutil.EMU_SO)
    h = ctypes.c_void_p()
    assert L.spex_executor_create(CFG.encode(), seed, b"t1,t2,t3", 1, ctypes.byref(h)) == 0
    if world:
        assert L.spex_executor_set_shard(h, rank, world) == 0
    t = _lib.Totals()
    assert L.spex_executor_run(h, 1, ctypes.byref(t)) == 0
    buf, n = ctypes.c_void_p(), ctypes.c_size_t()
    assert L.spex_executor_log(h, ctypes.byref(buf), ctypes.byref(n)) == 0
    log = ctypes.string_at(buf, n.value).decode()
    L.spex_free(buf)
    L.spex_executor_destroy(h)
    return log, t.queries


def _coupled_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_10195_b200.shard import query_block, reduce_report
    log, queries = _coupled_log(100, rank, world)
    lo, hi = query_block(queries, rank, world)
    mx, total = reduce_report(0.5 * (rank + 1), float(hi - lo), group=dist.group.WORLD)
    # every rank holds the same single-server log: gather its digest
    import hashlib
    import torch
    d = torch.tensor(list(hashlib.sha256(log.encode()).digest()), dtype=torch.uint8)
    ds = [torch.zeros_like(d) for _ in range(world)]
    dist.all_gather(ds, d)
    q.put((rank, log, lo, hi, mx, total, all(bool((x == ds[0]).all()) for x in ds)))
    dist.destroy_process_group()


@pytest.mark.skipif(not refutil.EMU_SO.exists(), reason="emulation library not built")
def test_two_rank_coupled_mode_over_gloo():
    """coupled mode: both ranks run the whole search (same seed) with their own
    query block set; the logs are identical to each other and to the unsharded
    run, the blocks partition the queries, the report sums to Q."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    ps = [ctx.Process(target=_coupled_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    full, nq = _coupled_log(100, 0, 0)
    assert nq == 4
    (_, l0, lo0, hi0, mx0, t0, same0), (_, l1, lo1, hi1, mx1, t1, same1) = res
    assert l0 == l1 == full and same0 and same1
    assert (lo0, hi0, lo1, hi1) == (0, 2, 2, 4)
    assert mx0 == mx1 == 1.0 and t0 == t1 == 4.0


@pytest.mark.skipif(not refutil.EMU_SO.exists(), reason="emulation library not built")
def test_set_shard_argument_errors():
    from paper_2605_10195_b200 import _lib
    from paper_2605_10195_b200.shard import query_block
    L = _lib.bind(refutil.EMU_SO)
    h = ctypes.c_void_p()
    assert L.spex_executor_create(CFG.encode(), 1, b"", 0, ctypes.byref(h)) == 0
    assert L.spex_executor_set_shard(h, 2, 2) != 0
    assert L.spex_executor_set_shard(h, -1, 2) != 0
    assert L.spex_executor_set_shard(h, 0, 0) != 0
    assert L.spex_executor_set_shard(h, 1, 3) == 0
    L.spex_executor_destroy(h)
    with pytest.raises(ValueError):
        query_block(8, 3, 3)
    blocks = [query_block(4096, r, 7) for r in range(7)]
    assert blocks[0][0] == 0 and blocks[-1][1] == 4096
    assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
