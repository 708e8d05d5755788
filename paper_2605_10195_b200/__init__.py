"""paper_2605_10195_b200 — B200-native SPEX frontier-expansion path.

Host-side mirror of the reference's whole-path entry points:

    Executor(cfg, run_seed, flags, trace).run() -> RunTotals   executor.hpp:50-58
    run_once(cfg, seed, flags) -> RunOutcome(totals, log)       experiment.hpp:27

with the reference's error convention: failures raise :class:`TotsimError`
whose ``code`` is the ``totsim::Errc`` name (errors.hpp:9-28). Every call goes
through the C-ABI (include/spex.h) into the sm_100a control kernel; there is
no CPU implementation behind this package.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import Any

from . import _lib

ERRC = [
    None,
    "UnknownParent",
    "ParentPruned",
    "NotSpeculative",
    "UnknownNode",
    "IllegalTransition",
    "ZeroVisits",
    "NoChildren",
    "EmptyRewards",
    "SearchComplete",
    "NothingExpandable",
    "UnknownSpeculation",
    "NegativeWeight",
    "EmptyTally",
    "EmptyBatch",
    "ConfigInvalid",
    "IncompleteLog",
    "IoFailure",
    "InvalidArgument",
]


class TotsimError(RuntimeError):
    """totsim::Error equivalent; ``code`` is the Errc name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERRC[status] if 0 < status < len(ERRC) else f"Device{status}"
        super().__init__(message)


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.lib().spex_last_error()
        raise TotsimError(rc, msg.decode() if msg else f"status {rc}")


@dataclass
class SpexFlags:
    """config.hpp:19-26."""

    t1: bool = False
    t2: bool = False
    t3: bool = False

    def any(self) -> bool:
        return self.t1 or self.t2 or self.t3

    def to_csv(self) -> str:
        return ",".join(n for n, on in (("t1", self.t1), ("t2", self.t2), ("t3", self.t3)) if on)

    def to_string(self) -> str:
        s = "+".join(n for n, on in (("t1", self.t1), ("t2", self.t2), ("t3", self.t3)) if on)
        return s or "baseline"

    @staticmethod
    def from_string(csv: str) -> "SpexFlags":
        f = SpexFlags()
        for item in csv.split(","):
            item = item.strip()
            if not item:
                continue
            if item not in ("t1", "t2", "t3"):
                raise TotsimError(15, f"unknown flag: {item}")
            setattr(f, item, True)
        return f


@dataclass
class RunTotals:
    makespan: float = 0.0
    generated_tokens: int = 0
    committed_tokens: int = 0
    reused_tokens: int = 0
    wasted_tokens: int = 0
    hits: list = field(default_factory=lambda: [0] * 9)
    misses: list = field(default_factory=lambda: [0] * 9)
    queries: int = 0
    correct_votes: int = 0
    early_terminated: int = 0

    def useful_tokens(self) -> int:
        return self.committed_tokens + self.reused_tokens


@dataclass
class RunOutcome:
    totals: RunTotals
    log: list


def _cfg_text(cfg: Any) -> str:
    if isinstance(cfg, (bytes, str)):
        return cfg.decode() if isinstance(cfg, bytes) else cfg
    return json.dumps(cfg)


def canonical_config(cfg: Any) -> dict:
    """ExperimentConfig::from_json(...).to_json() (strict; ConfigInvalid on unknown keys)."""
    L = _lib.lib()
    out = ctypes.c_void_p()
    _check(L.spex_canonical_config(_cfg_text(cfg).encode(), ctypes.byref(out)))
    try:
        return json.loads(ctypes.string_at(out.value).decode())
    finally:
        L.spex_free(out)


def device_ok() -> bool:
    return bool(_lib.lib().spex_device_ok())


class Executor:
    """Executor(cfg, run_seed, flags, trace) (executor.hpp:43-62). ``flags`` None
    uses the config's own run.flags."""

    def __init__(self, cfg: Any, run_seed: int, flags: SpexFlags | str | None = None,
                 trace: bool = True, device: int = 0):
        L = _lib.lib()
        if not L.spex_device_ok():
            raise RuntimeError("no sm_100 CUDA device: the SPEX B200 path has no CPU fallback")
        if isinstance(flags, SpexFlags):
            fcsv = flags.to_csv().encode()
        elif isinstance(flags, str):
            fcsv = flags.encode()
        else:
            fcsv = None
        self._L = L
        self._trace = trace
        h = ctypes.c_void_p()
        _check(L.spex_executor_create(_cfg_text(cfg).encode(), int(run_seed), fcsv, device, ctypes.byref(h)))
        self._h = h

    def run(self) -> RunTotals:
        t = _lib.Totals()
        _check(self._L.spex_executor_run(self._h, 1 if self._trace else 0, ctypes.byref(t)))
        d = t.as_dict()
        return RunTotals(**d)

    def step(self, iterations: int = 1) -> tuple:
        """The fused device frontier step: run up to ``iterations`` iterations
        of the consumer loop (executor.cpp:785-807; 0 = to the end) on the
        device. Returns (done, event-log lines of this call)."""
        done = ctypes.c_int()
        out = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(self._L.spex_frontier_step(self._h, int(iterations), ctypes.byref(done), ctypes.byref(out),
                                          ctypes.byref(n)))
        try:
            lines = ctypes.string_at(out.value, n.value).decode().splitlines() if out.value else []
        finally:
            self._L.spex_free(out)
        return bool(done.value), lines

    def log_lines(self) -> list:
        out = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(self._L.spex_executor_log(self._h, ctypes.byref(out), ctypes.byref(n)))
        try:
            return ctypes.string_at(out.value, n.value).decode().splitlines()
        finally:
            self._L.spex_free(out)

    def stats(self) -> dict:
        s = _lib.Stats()
        _check(self._L.spex_executor_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def set_model(self, policy: str = "small_policy", prm: str = "small_prm", weight_seed: int = 1,
                  record_outputs: bool = False) -> None:
        """Attach the policy/PRM forward: every scheduled decode row and every
        completed thought runs through the models on the device."""
        _check(self._L.spex_executor_set_model(self._h, policy.encode(), (prm or "").encode(), int(weight_seed),
                                               1 if record_outputs else 0))

    def set_shard(self, rank: int, world: int) -> None:
        """Run the model forward only for this rank's query block
        [Q*rank/world, Q*(rank+1)/world); the search itself stays whole, so
        every rank's decisions and log equal the single-server reference's."""
        _check(self._L.spex_executor_set_shard(self._h, int(rank), int(world)))

    def set_split(self, rank: int, world: int, outboxes, epoch: int) -> None:
        """Split mode (shard.Outboxes builds ``outboxes``): this executor is
        rank ``rank`` of a ``world``-rank job — its query block with its own
        engine and clock, T2 budgets allocated over every rank's candidates.
        ``epoch`` >= 1 is the run id, the same on every rank."""
        arr = (ctypes.c_void_p * int(world))(*outboxes)
        _check(self._L.spex_executor_set_split(self._h, int(rank), int(world), arr, int(epoch)))

    def emulate_split(self, rank: int, world: int) -> None:
        """One GPU standing in for ``world``: this executor runs rank ``rank``
        (model included) while the other ranks' control runs beside it on the
        same device; decisions and this rank's work are the multi-GPU run's."""
        _check(self._L.spex_executor_emulate_split(self._h, int(rank), int(world)))

    def split_stats(self) -> dict:
        r, w = ctypes.c_longlong(), ctypes.c_double()
        _check(self._L.spex_executor_split_stats(self._h, ctypes.byref(r), ctypes.byref(w)))
        return {"rounds": r.value, "wait_ms": w.value}

    def set_kv_pages(self, pages: int) -> None:
        """Tree-KV pool size in pages of 16 tokens (0: the default, 70% of free HBM)."""
        _check(self._L.spex_executor_set_kv_pages(self._h, int(pages)))

    def set_reward_source(self, source: str) -> None:
        """"oracle": rewards from the content oracle (the reference's RewardOracle);
        "prm": rewards are the PRM's scores, awaited on device (model mode)."""
        if source not in ("oracle", "prm"):
            raise ValueError("reward source is 'oracle' or 'prm'")
        _check(self._L.spex_executor_set_reward_source(self._h, 1 if source == "prm" else 0))

    def query_wall_ms(self) -> tuple:
        """(per-query device wall-clock latency in ms, ms the control waited for PRM scores)."""
        n = ctypes.c_int()
        w = ctypes.c_double()
        _check(self._L.spex_executor_query_wall_ms(self._h, None, 0, ctypes.byref(n), ctypes.byref(w)))
        buf = (ctypes.c_double * max(n.value, 1))()
        _check(self._L.spex_executor_query_wall_ms(self._h, buf, n.value, ctypes.byref(n), ctypes.byref(w)))
        return list(buf[: n.value]), w.value

    def kv_stats(self) -> dict:
        s = _lib.KvStats()
        _check(self._L.spex_executor_kv_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def model_stats(self) -> dict:
        s = _lib.ModelStats()
        _check(self._L.spex_executor_model_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def decode_outputs(self) -> list:
        n = ctypes.c_longlong()
        _check(self._L.spex_executor_decode_outputs(self._h, None, 0, ctypes.byref(n)))
        buf = (_lib.DecodeOut * max(n.value, 1))()
        _check(self._L.spex_executor_decode_outputs(self._h, buf, n.value, ctypes.byref(n)))
        return [(o.q, o.node, o.pos, o.argmax, o.lse, o.logit_sum) for o in buf[: n.value]]

    def prm_outputs(self) -> list:
        n = ctypes.c_longlong()
        _check(self._L.spex_executor_prm_outputs(self._h, None, 0, ctypes.byref(n)))
        buf = (_lib.PrmOut * max(n.value, 1))()
        _check(self._L.spex_executor_prm_outputs(self._h, buf, n.value, ctypes.byref(n)))
        return [(o.q, o.node, o.score) for o in buf[: n.value]]

    def query_finish_times(self) -> list:
        """Virtual finish time of every query (its search latency when all are admitted at t=0)."""
        n = ctypes.c_int()
        cap = 1 << 16
        buf = (ctypes.c_double * cap)()
        _check(self._L.spex_executor_query_finish(self._h, buf, cap, ctypes.byref(n)))
        return list(buf[: min(n.value, cap)])

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.spex_executor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_once(cfg: Any, seed: int, flags: SpexFlags | str | None = None) -> RunOutcome:
    """run_once (experiment.cpp:23-30): a traced run with totals and the log."""
    ex = Executor(cfg, seed, flags, trace=True)
    try:
        totals = ex.run()
        return RunOutcome(totals=totals, log=ex.log_lines())
    finally:
        ex.close()


def run(cfg: Any, seed: int, flags: SpexFlags | str | None = None, on_event=None, chunk: int = 4096) -> RunTotals:
    """spex_run: the whole run stepped on the device ``chunk`` consumer-loop
    iterations at a time, each event-log line passed to ``on_event(line)`` as
    it is produced (the run_once log, streamed)."""
    L = _lib.lib()
    if not L.spex_device_ok():
        raise RuntimeError("no sm_100 CUDA device: the SPEX B200 path has no CPU fallback")
    fcsv = flags.to_csv().encode() if isinstance(flags, SpexFlags) else (flags.encode() if isinstance(flags, str)
                                                                          else None)
    cb = _lib.TRACE_CB(lambda line, n, user: on_event(line[:n].decode()) if on_event else None)
    t = _lib.Totals()
    _check(L.spex_run(_cfg_text(cfg).encode(), int(seed), fcsv, cb, None, int(chunk), ctypes.byref(t)))
    return RunTotals(**t.as_dict())


def run_batch(cfg: Any, seeds, flags: SpexFlags | str | None = None, device: int = 0):
    """Independent searches of one config, one per seed, in ONE launch of the
    control kernel (one CTA per search; control only, no model). The device
    analog of run_experiment_full's loop over repetitions (experiment.cpp:61-78).
    Returns (list of RunTotals, device milliseconds of the launch)."""
    L = _lib.lib()
    seeds = list(seeds)
    n = len(seeds)
    arr = (ctypes.c_uint64 * n)(*seeds)
    tots = (_lib.Totals * n)()
    ms = ctypes.c_double()
    if isinstance(flags, SpexFlags):
        fcsv = flags.to_csv().encode()
    elif isinstance(flags, str):
        fcsv = flags.encode()
    else:
        fcsv = None
    _check(L.spex_run_batch(_cfg_text(cfg).encode(), arr, n, fcsv, device, tots, ctypes.byref(ms)))
    return [RunTotals(**t.as_dict()) for t in tots], ms.value


def score_batch(prm_shape: str, weight_seed: int, sequences, device: int = 0) -> list:
    """PRM scores of standalone token sequences (spex_score_batch): the value
    head at each sequence's last token, with the PRM weights
    Executor.set_model gives for ``weight_seed``."""
    L = _lib.lib()
    if not L.spex_device_ok():
        raise RuntimeError("no sm_100 CUDA device: the SPEX B200 path has no CPU fallback")
    seqs = [list(map(int, s)) for s in sequences]
    flat = [t for s in seqs for t in s]
    offs = [0]
    for s in seqs:
        offs.append(offs[-1] + len(s))
    toks = (ctypes.c_int32 * max(1, len(flat)))(*flat)
    off = (ctypes.c_int64 * len(offs))(*offs)
    out = (ctypes.c_float * max(1, len(seqs)))()
    _check(L.spex_score_batch(prm_shape.encode(), int(weight_seed), toks, off, len(seqs), out, device))
    return [out[i] for i in range(len(seqs))]


def split_run(cfg: Any, seed: int, world: int, flags: SpexFlags | str | None = None, trace: bool = True,
              device: int = 0) -> list:
    """Every rank of one split job (shard.py) on one device, as CTAs of one
    control launch (control only). One dict per rank: log, rounds, stats."""
    from . import shard
    if isinstance(flags, SpexFlags):
        fcsv = flags.to_csv()
    else:
        fcsv = flags
    L = _lib.lib()
    if not L.spex_device_ok():
        raise RuntimeError("no sm_100 CUDA device: the SPEX B200 path has no CPU fallback")
    return shard.split_run(L, _cfg_text(cfg), seed, world, fcsv, trace, device)


__all__ = [
    "Executor",
    "RunOutcome",
    "RunTotals",
    "SpexFlags",
    "TotsimError",
    "canonical_config",
    "device_ok",
    "run",
    "run_batch",
    "run_once",
    "score_batch",
    "split_run",
]
