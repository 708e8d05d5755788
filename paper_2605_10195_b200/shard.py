"""Query sharding across GPUs, two modes.

independent: each rank owns a disjoint query set — a whole search with run
seed ``base + rank`` (generate_workload derives every query seed from the run
seed, sim.cpp:177-180) — so no KV, tree or schedule state crosses GPUs and the
data path needs no collective (weak scaling).

coupled: ONE search of Q queries as the reference's single server runs it.
Every rank runs the same control kernel (one SM) over all Q queries, so the
virtual clock, the global T2 budget allocation (executor.cpp:705-740) and the
event log are the reference's on every rank with no exchange at all; rank r
runs the model work (policy decode, tree KV, PRM) of query block
``query_block(Q, r, W)`` only (``Executor.set_shard``), strong scaling. The
exchange SURVEY.md §8e prices for a split control (an allgather of per-query
gains per scheduling round plus an allreduce of (B, U) per engine epoch, ~1e5
collectives per search) is replaced by recomputing the ~1 SM of control.

Ranks meet only to report: max over ranks of the step time, sum of queries
(owned queries in coupled mode, so the sum is Q)."""

from __future__ import annotations


def query_block(n_queries: int, rank: int, world: int) -> tuple:
    """[lo, hi) of rank's query block (spex_executor_set_shard's split)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    return n_queries * rank // world, n_queries * (rank + 1) // world


def shard_seed(base_seed: int, rank: int) -> int:
    return base_seed + rank


def reduce_report(step_seconds: float, queries: float, group=None):
    """Returns (max step seconds over ranks, total queries)."""
    if group is None:
        return step_seconds, queries
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([step_seconds], dtype=torch.float64, device=dev)
    q = torch.tensor([queries], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(q, op=dist.ReduceOp.SUM)
    return float(t.item()), float(q.item())
