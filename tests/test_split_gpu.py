"""GPU: the split multi-GPU mode on the sm_100a control kernel.
Every rank of a job runs as one CTA of one launch on this B200 (the exchange
spins on the other ranks, so they must be co-resident), or as one process per
rank with CUDA-IPC outboxes; each rank's event log must equal, byte for byte,
the split oracle's (oracle/ref_split.cpp: the reference's own executor, one
thread per rank, coupled by the same T2 budget exchange)."""
import hashlib
import json
import os
import socket
from pathlib import Path

import pytest

import paper_2605_10195_b200 as spex
from paper_2605_10195_b200 import shard
from tests import refutil

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CFG = ROOT / "configs"
GOLDEN = ROOT / "tests" / "golden"
needs_oracle = pytest.mark.skipif(refutil.ref_split_lib() is None, reason="oracle/_ref not built")


def _digest(lines):
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()


CASES = [(n, w) for n in ("c1_rebase_w4_q16", "c3_rstar_w4_q512") for w in (1, 2, 3, 4, 8)]
CASES += [("c3_rstar_w4_q512_t1t3", 8)]  # the literal config 3 (no T2: blocks without exchange)


@needs_oracle
@pytest.mark.parametrize("name,W", CASES)
def test_split_matches_oracle(name, W):
    cfg = (CFG / f"{name}.json").read_text()
    ref, rounds = refutil.ref_split_log(cfg, 1, None, W)
    got = spex.split_run(cfg, 1, W)
    assert [g["rounds"] for g in got] == (rounds if W > 1 else [0])
    for r in range(W):
        assert got[r]["log"] == ref[r], (name, W, r, refutil.compare_logs(ref[r], got[r]["log"]))


@needs_oracle
@pytest.mark.parametrize("name,cfg,seed,flags", refutil.split_configs())
def test_split_sweep(name, cfg, seed, flags):
    for W in (2, 5):
        ref, rounds = refutil.ref_split_log(cfg, seed, flags, W)
        got = spex.split_run(cfg, seed, W, flags)
        assert [g["rounds"] for g in got] == rounds
        for r in range(W):
            assert got[r]["log"] == ref[r], (name, W, r, refutil.compare_logs(ref[r], got[r]["log"]))


def test_split_c4_w8_golden_digest():
    """Config 4 (rest_hybrid, 4096 queries, T1+T2+T3) over 8 ranks against the
    committed oracle digest (tests/golden/make_split_digest.py)."""
    gold = json.loads((GOLDEN / "split_c4_w8_digest.json").read_text())
    cfg = (CFG / "c4_rest_w4_q4096.json").read_text()
    got = spex.split_run(cfg, gold["seed"], gold["world"])
    assert [g["rounds"] for g in got] == gold["rounds"]
    assert [len(g["log"]) for g in got] == gold["lines"]
    assert [_digest(g["log"]) for g in got] == gold["sha256"]


@needs_oracle
@pytest.mark.parametrize("W", [2, 4])
def test_split_c4_matches_oracle(W):
    cfg = (CFG / "c4_rest_w4_q4096.json").read_text()
    ref, rounds = refutil.ref_split_log(cfg, 1, None, W)
    got = spex.split_run(cfg, 1, W)
    assert [g["rounds"] for g in got] == rounds
    for r in range(W):
        assert got[r]["log"] == ref[r], (W, r, refutil.compare_logs(ref[r], got[r]["log"]))


# ------------------------------------- one process per rank, CUDA IPC outboxes
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, cfg, seed, out_dir, model):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_10195_b200 import _lib
        L = _lib.lib()
        boxes = shard.Outboxes(L, rank, world, json.loads(cfg)["run"]["n_queries"], kind="cuda")
        out = {}
        for epoch in (1, 2):  # two runs through the same outboxes (epoch-tagged flags, no reset)
            ex = spex.Executor(cfg, seed, None, trace=True)
            if model:
                ex.set_model("small_policy", "small_prm", 1)
                ex.set_kv_pages(1 << 15)  # two processes share this GPU
            ex.set_split(rank, world, boxes.pointers, epoch)
            dist.barrier()
            ex.run()
            out[epoch] = {"log": ex.log_lines(), **ex.split_stats()}
            if model:
                out[epoch]["model"] = ex.model_stats()
            ex.close()
        (Path(out_dir) / f"rank{rank}.json").write_text(json.dumps(out))
        dist.barrier()
        boxes.close()
    finally:
        dist.destroy_process_group()


@needs_oracle
@pytest.mark.timeout(600)
@pytest.mark.parametrize("model", [False, True], ids=["control", "model"])
def test_split_one_process_per_rank_ipc(tmp_path, model):
    """Two processes (the multi-GPU launch shape; here both on this GPU,
    time-sliced): CUDA-IPC outboxes, handles exchanged over gloo, the control
    kernels exchanging through peer memory; with the small policy + PRM forward
    attached in the second case."""
    import torch.multiprocessing as mp
    cfg = (CFG / "c1_rebase_w4_q16.json").read_text()
    W = 2
    mp.start_processes(_rank_main, args=(W, _free_port(), cfg, 1, str(tmp_path), model), nprocs=W, join=True,
                       start_method="spawn")
    ref, rounds = refutil.ref_split_log(cfg, 1, None, W)
    for r in range(W):
        got = json.loads((tmp_path / f"rank{r}.json").read_text())
        for epoch in ("1", "2"):
            assert got[epoch]["rounds"] == rounds[r]
            assert got[epoch]["log"] == ref[r], (r, epoch, refutil.compare_logs(ref[r], got[epoch]["log"]))
            if model:
                assert got[epoch]["model"]["decode_rows"] > 0


@needs_oracle
@pytest.mark.parametrize("W,rank", [(2, 1), (4, 0), (4, 3)])
def test_emulated_rank_matches_oracle(W, rank):
    """One rank live (with the small policy + PRM forward), the others' control
    beside it on this GPU: the rank's log is the split oracle's."""
    cfg = (CFG / "c3_rstar_w4_q512.json").read_text()
    ref, rounds = refutil.ref_split_log(cfg, 1, None, W)
    ex = spex.Executor(cfg, 1, None, trace=True)
    ex.set_model("small_policy", "small_prm", 1)
    ex.emulate_split(rank, W)
    ex.run()
    assert ex.split_stats()["rounds"] == rounds[rank]
    assert ex.log_lines() == ref[rank]
    assert ex.model_stats()["decode_rows"] > 0
    ex.close()


def _random_split_cases():
    """Random configurations (tests/refutil.random_configs) with T2 forced on,
    so every case exercises the budget exchange, at 2-4 ranks."""
    out = []
    for k, (name, cfg, seed, flags) in enumerate(refutil.random_configs(n=40, seed=77)):
        c = json.loads(cfg)
        if c["run"]["n_queries"] < 2:
            continue
        fl = ",".join(sorted(set((flags.split(",") if flags else []) + ["t1", "t2"])))
        out.append((name, json.dumps(c), seed, fl, 2 + k % 3))
    return out[:24]


@needs_oracle
@pytest.mark.parametrize("name,cfg,seed,flags,W", _random_split_cases())
def test_split_random_configs(name, cfg, seed, flags, W):
    W = min(W, json.loads(cfg)["run"]["n_queries"])
    ref, rounds = refutil.ref_split_log(cfg, seed, flags, W)
    got = spex.split_run(cfg, seed, W, flags)
    assert [g["rounds"] for g in got] == rounds
    for r in range(W):
        assert got[r]["log"] == ref[r], (name, W, r, refutil.compare_logs(ref[r], got[r]["log"]))
