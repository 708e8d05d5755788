"""CPU: the split multi-GPU mode (shard.py) — each rank owns a
query block with its own engine and clock; the only exchange is T2's budget
round. The oracle is the reference's own executor in one thread per rank
(oracle/ref_split.cpp); the device control code runs here in the test-only
emulation library (ranks = host threads, or processes over gloo with shared-
memory outboxes). The sm_100a kernel is checked in tests/test_split_gpu.py."""
import ctypes
import hashlib
import json
import os
import socket
from pathlib import Path

import pytest

from paper_2605_10195_b200 import _lib, shard
from tests import refutil

ROOT = Path(__file__).resolve().parents[1]
CFG = ROOT / "configs"
GOLDEN = ROOT / "tests" / "golden"

needs_oracle = pytest.mark.skipif(refutil.ref_split_lib() is None or refutil.ref_lib() is None,
                                  reason="oracle/_ref not built")


def emu():
    if not refutil.EMU_SO.exists():
        pytest.skip("emulation library not built (make -C paper_2605_10195_b200/csrc emu)")
    return _lib.bind(refutil.EMU_SO)


@needs_oracle
@pytest.mark.parametrize("name", ["c1_rebase_w4_q16", "c3_rstar_w4_q512"])
def test_oracle_world1_is_the_reference(name):
    cfg = (CFG / f"{name}.json").read_text()
    logs, _ = refutil.ref_split_log(cfg, 1, None, 1)
    assert logs[0] == refutil.ref_run_log(cfg, 1, None)


@needs_oracle
def test_oracle_ranks_keep_the_jobs_queries():
    """Rank r's local query q is the job's query lo(r) + q: same seed as in
    the single-server run (generate_workload, sim.cpp:177-180)."""
    cfg = (CFG / "c1_rebase_w4_q16.json").read_text()
    single = [json.loads(x) for x in refutil.ref_run_log(cfg, 1, None)]
    seeds = {e["q"]: e["seed"] for e in single if e["ev"] == "admit"}
    W = 3
    logs, _ = refutil.ref_split_log(cfg, 1, None, W)
    for r, log in enumerate(logs):
        lo, hi = shard.query_block(16, r, W)
        recs = [json.loads(x) for x in log]
        assert recs[0]["config"]["run"]["n_queries"] == hi - lo
        adm = {e["q"]: e["seed"] for e in recs if e["ev"] == "admit"}
        assert adm == {q - lo: seeds[q] for q in range(lo, hi)}


@needs_oracle
@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("name", ["c1_rebase_w4_q16", "c3_rstar_w4_q512"])
def test_emulation_split_matches_oracle(name, W):
    L = emu()
    cfg = (CFG / f"{name}.json").read_text()
    ref, rounds = refutil.ref_split_log(cfg, 1, None, W)
    got = shard.split_run(L, cfg, 1, W)
    assert [g["rounds"] for g in got] == rounds
    assert sum(rounds) > 0  # the exchange ran (T2 configs)
    for r in range(W):
        assert got[r]["log"] == ref[r], (name, W, r, refutil.compare_logs(ref[r], got[r]["log"]))


@needs_oracle
@pytest.mark.parametrize("name,cfg,seed,flags", refutil.split_configs())
def test_emulation_split_sweep(name, cfg, seed, flags):
    L = emu()
    for W in (2, 5):
        ref, rounds = refutil.ref_split_log(cfg, seed, flags, W)
        got = shard.split_run(L, cfg, seed, W, flags)
        assert [g["rounds"] for g in got] == rounds
        for r in range(W):
            assert got[r]["log"] == ref[r], (name, W, r, refutil.compare_logs(ref[r], got[r]["log"]))


def _digest(lines):
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()


def test_emulation_split_c4_w8_matches_golden_digest():
    """Config 4 (rest_hybrid, 4096 queries, T1+T2+T3) over 8 ranks: the rank
    logs' SHA-256 pinned from the oracle (tests/golden/make_split_digest.py)."""
    L = emu()
    gold = json.loads((GOLDEN / "split_c4_w8_digest.json").read_text())
    cfg = (CFG / "c4_rest_w4_q4096.json").read_text()
    got = shard.split_run(L, cfg, gold["seed"], gold["world"])
    assert [g["rounds"] for g in got] == gold["rounds"]
    assert [_digest(g["log"]) for g in got] == gold["sha256"]


def test_split_argument_checks():
    L = emu()
    assert L.spex_split_outbox_bytes(16, 0) == -1
    assert L.spex_split_outbox_bytes(4, 5) == -1
    assert L.spex_split_outbox_bytes(16, 65) == -1
    assert L.spex_split_outbox_bytes(4096, 8) > 512 * 12
    cfg = (CFG / "c1_rebase_w4_q16.json").read_text()
    h = ctypes.c_void_p()
    assert L.spex_executor_create(cfg.encode(), 1, None, 0, ctypes.byref(h)) == 0
    try:
        boxes = (ctypes.c_void_p * 2)()
        assert L.spex_executor_set_split(h, 2, 2, boxes, 1) != 0           # rank out of range
        assert L.spex_executor_set_split(h, 0, 2, None, 1) != 0            # no outboxes
        assert L.spex_executor_set_split(h, 0, 17, boxes, 1) != 0          # more ranks than queries
        assert L.spex_executor_set_shard(h, 0, 2) == 0
        assert L.spex_executor_set_split(h, 0, 2, boxes, 1) != 0           # coupled shard already set
    finally:
        L.spex_executor_destroy(h)


# ------------------------------------------------ one process per rank (gloo)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, cfg, seed, out_dir, tag):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = _lib.bind(refutil.EMU_SO)
        boxes = shard.Outboxes(L, rank, world, json.loads(cfg)["run"]["n_queries"], kind="shm", tag=tag)
        dist.barrier()
        h = ctypes.c_void_p()
        assert L.spex_executor_create(cfg.encode(), seed, None, 0, ctypes.byref(h)) == 0
        boxes.attach(h, epoch=1)
        t = _lib.Totals()
        rc = L.spex_executor_run(h, 1, ctypes.byref(t))
        assert rc == 0, L.spex_last_error()
        res = shard.rank_result(L, h)
        L.spex_executor_destroy(h)
        (Path(out_dir) / f"rank{rank}.json").write_text(json.dumps({"log": res["log"], "rounds": res["rounds"]}))
        dist.barrier()
        boxes.close()
    finally:
        dist.destroy_process_group()


@needs_oracle
def test_split_one_process_per_rank_gloo(tmp_path):
    """World size 2 over gloo: each process owns its outbox (shared memory for
    the CPU emulation; CUDA IPC on GPUs), the handles go through
    all_gather_object, and the control loops exchange through the outboxes."""
    emu()
    import torch.multiprocessing as mp
    cfg = (CFG / "c1_rebase_w4_q16.json").read_text()
    W = 2
    mp.start_processes(_rank_main, args=(W, _free_port(), cfg, 1, str(tmp_path), f"spex{os.getpid()}"), nprocs=W,
                       join=True, start_method="spawn")
    ref, rounds = refutil.ref_split_log(cfg, 1, None, W)
    for r in range(W):
        got = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert got["rounds"] == rounds[r]
        assert got["log"] == ref[r]


def _rank_fail_main(rank, world, port, out_dir, tag):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = _lib.bind(refutil.EMU_SO)
        kind = "shm" if rank == 0 else "no-such-kind"  # rank 1 cannot set up its outbox
        try:
            shard.Outboxes(L, rank, world, 16, kind=kind, tag=tag)
            res = "ok"
        except shard.SplitUnavailable as e:
            res = "unavailable: " + str(e)
        (Path(out_dir) / f"rank{rank}.txt").write_text(res)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_split_setup_failure_is_agreed_by_every_rank(tmp_path):
    """One rank failing to set up its outbox makes every rank raise
    SplitUnavailable (bench.py then runs independent shards on all ranks)
    instead of leaving the others waiting in a collective."""
    emu()
    import torch.multiprocessing as mp
    mp.start_processes(_rank_fail_main, args=(2, _free_port(), str(tmp_path), f"spexf{os.getpid()}"), nprocs=2,
                       join=True, start_method="spawn")
    for r in range(2):
        msg = (tmp_path / f"rank{r}.txt").read_text()
        assert msg.startswith("unavailable") and "rank 1" in msg, msg


@needs_oracle
def test_emulation_split_random_configs():
    """The GPU file's random T2 cases (tests/test_split_gpu.py) in the emulation."""
    from tests.test_split_gpu import _random_split_cases
    L = emu()
    for name, cfg, seed, flags, W in _random_split_cases():
        W = min(W, json.loads(cfg)["run"]["n_queries"])
        ref, rounds = refutil.ref_split_log(cfg, seed, flags, W)
        got = shard.split_run(L, cfg, seed, W, flags)
        assert [g["rounds"] for g in got] == rounds, name
        for r in range(W):
            assert got[r]["log"] == ref[r], (name, W, r, refutil.compare_logs(ref[r], got[r]["log"]))
