"""Query sharding across GPUs: each rank owns a disjoint query
set — here a whole search with run seed ``base + rank`` (generate_workload
derives every query seed from the run seed, sim.cpp:177-180) — so no KV, tree
or schedule state crosses GPUs and the data path needs no collective. Ranks
meet only to report: max over ranks of the step time, sum of queries."""
from __future__ import annotations


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
