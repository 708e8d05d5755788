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
