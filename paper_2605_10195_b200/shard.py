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

split (north_star's data path): ONE job of Q queries; rank r owns query block
``query_block(Q, r, W)`` outright — its own control kernel, decode engine,
virtual clock and tree KV — and the ranks exchange only T2's per-query gains:
the k-th budget allocation of every rank is one round over every rank's
candidates (``Executor.set_split``; the control kernels read each other's
outboxes over NVLink, no host round trip). Oracle:
oracle/ref_split.cpp.

Ranks meet only to report: max over ranks of the step time, sum of queries
(owned queries in coupled and split mode, so the sum is Q)."""

from __future__ import annotations

import ctypes



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


def split_run(L, cfg_text: str, seed: int, world: int, flags_csv: str | None = None, trace: bool = True,
              device: int = 0) -> list:
    """Every rank of one split job on ONE device, CTA r = rank r of one control
    launch (spex_split_run; control only). ``L`` is a bound library (the
    product, or the test-only emulation, where the ranks are host threads).
    Returns one dict per rank: totals, log lines, exchange rounds, wait ms."""
    from . import _lib
    out = (ctypes.c_void_p * world)()
    rc = L.spex_split_run(cfg_text.encode(), int(seed), None if flags_csv is None else flags_csv.encode(), world,
                          device, 1 if trace else 0, out)
    if rc:
        raise RuntimeError(f"spex_split_run: {L.spex_last_error().decode()}")
    res = []
    try:
        for r in range(world):
            res.append(rank_result(L, out[r], trace))
    finally:
        for r in range(world):
            L.spex_executor_destroy(out[r])
    return res


def rank_result(L, h, trace: bool = True) -> dict:
    """Totals, log, exchange rounds and wait time of one rank's executor."""
    from . import _lib
    t = _lib.Totals()
    st = _lib.Stats()
    L.spex_executor_stats(h, ctypes.byref(st))
    rounds, wait = ctypes.c_longlong(), ctypes.c_double()
    L.spex_executor_split_stats(h, ctypes.byref(rounds), ctypes.byref(wait))
    log = []
    if trace:
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        if L.spex_executor_log(h, ctypes.byref(p), ctypes.byref(n)) == 0:
            log = ctypes.string_at(p.value, n.value).decode().splitlines()
            L.spex_free(p)
    return {"log": log, "rounds": rounds.value, "wait_ms": wait.value, "stats": st.as_dict()}


class SplitUnavailable(RuntimeError):
    """The outboxes could not be set up on some rank (raised on every rank)."""


class Outboxes:
    """The ranks' split-mode outboxes, one process per rank.

    kind "cuda": this rank's outbox in its GPU's HBM (spex_split_outbox_alloc),
    the others mapped through CUDA IPC handles (peer access over NVLink).
    kind "shm": host shared memory (the test-only emulation library, whose
    control runs on the CPU). The handles are exchanged with
    torch.distributed.all_gather_object over ``group`` (gloo or NCCL); nothing
    else of the exchange goes through the host."""

    def __init__(self, L, rank: int, world: int, n_queries_job: int, device: int = 0, group=None,
                 kind: str = "cuda", tag: str = "spex"):
        import torch.distributed as dist
        self._L, self.rank, self.world, self.kind = L, rank, world, kind
        nbytes = L.spex_split_outbox_bytes(n_queries_job, world)
        if nbytes < 0:
            raise ValueError("split: need 1 <= world <= min(64, n_queries)")
        self._shm = []
        self._opened = []
        self._own = None
        mine, err = None, ""
        try:
            if kind == "cuda":
                own = ctypes.c_void_p()
                handle = ctypes.create_string_buffer(64)
                if L.spex_split_outbox_alloc(device, nbytes, ctypes.byref(own), handle):
                    raise RuntimeError(L.spex_last_error().decode())
                self._own = own.value
                mine = bytes(handle.raw)
            elif kind == "shm":
                from multiprocessing import shared_memory
                shm = shared_memory.SharedMemory(create=True, size=int(nbytes), name=f"{tag}_{rank}_{world}")
                shm.buf[:nbytes] = bytes(nbytes)
                self._shm.append(shm)
                self._own = ctypes.addressof(ctypes.c_char.from_buffer(shm.buf))
                mine = shm.name
            else:
                raise ValueError("kind is 'cuda' or 'shm'")
        except Exception as e:  # every rank learns it below, so all ranks take the same path
            err = f"rank {rank}: {e}"
        handles = [None] * world
        dist.all_gather_object(handles, (mine, err), group=group)
        errs = [e for _, e in handles if e]
        if errs:
            self.close()
            raise SplitUnavailable("; ".join(errs))
        ptrs, err = [], ""
        try:
            for s, (h, _) in enumerate(handles):
                if s == rank:
                    ptrs.append(self._own)
                elif kind == "cuda":
                    p = ctypes.c_void_p()
                    if L.spex_split_outbox_open(device, h, ctypes.byref(p)):
                        raise RuntimeError(L.spex_last_error().decode())
                    self._opened.append(p.value)
                    ptrs.append(p.value)
                else:
                    from multiprocessing import shared_memory
                    peer = shared_memory.SharedMemory(name=h)
                    self._shm.append(peer)
                    ptrs.append(ctypes.addressof(ctypes.c_char.from_buffer(peer.buf)))
        except Exception as e:
            err = f"rank {rank}: {e}"
        oks = [None] * world
        dist.all_gather_object(oks, err, group=group)
        if any(oks):
            self.close()
            raise SplitUnavailable("; ".join(e for e in oks if e))
        self.pointers = ptrs

    def attach(self, h, epoch: int) -> None:
        """Make executor handle ``h`` this rank of the job for run ``epoch``
        (>= 1, the same on every rank, new for each run)."""
        arr = (ctypes.c_void_p * self.world)(*self.pointers)
        if self._L.spex_executor_set_split(h, self.rank, self.world, arr, int(epoch)):
            raise RuntimeError(self._L.spex_last_error().decode())

    def close(self) -> None:
        for p in self._opened:
            self._L.spex_split_outbox_close(ctypes.c_void_p(p))
        self._opened = []
        if self.kind == "cuda" and self._own:
            self._L.spex_split_outbox_free(ctypes.c_void_p(self._own))
        self._own = None
        for i, shm in enumerate(self._shm):
            try:
                shm.close()
                if i == 0:
                    shm.unlink()
            except Exception:
                pass
        self._shm = []
