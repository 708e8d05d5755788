#!/usr/bin/env python
"""bench.py — ToT queries/sec of the B200 frontier-expansion path (BASELINE.json metric).

One *step* = one complete batched ToT search over the config's query batch on
one GPU: the device-resident control kernel (decode engine, rewards, REBASE /
REST / RSTAR drivers, T1 speculation, T2 budgets, T3 termination) plus the real
policy decode of every scheduled row (K1 tree attention, projections, LM-head
epilogue) and PRM scoring of every completed thought (K4). The workload is
BASELINE config 2 (rebase_bfs, width 16, T1, 256 queries) with the builder's
mid-size random-init policy/PRM (the config names no model).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs one process per GPU (torchrun): each rank searches a disjoint query
set (run seed + rank; weak scaling, no data-path collective); rank 0 prints the
line with the max-over-ranks time. `--impl reference` times the reference's own
CPU implementation (oracle/_ref, compiled from the reference sources) on all
host cores for the same config and metric.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# concurrent searches (control_only) each run on their own stream: give the
# device 32 hardware queues instead of 8 so independent control CTAs do not
# serialise behind each other (read at CUDA initialisation)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from paper_2605_10195_b200.shard import query_block, shard_seed  # noqa: E402

DEFAULT_CONFIG = "c2_rebase_w16_q256"
PEAKS = ROOT / "MEASURED_PEAKS.json"
PROFILE_TRAFFIC = ROOT / "profiles" / "k1_traffic.json"
HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--policy", default="mid_policy")
    ap.add_argument("--prm", default="mid_prm")
    ap.add_argument("--cpu-sample-runs", type=int, default=4)
    ap.add_argument("--sharding", default="split", choices=["split", "independent", "coupled"],
                    help="split (north_star): ONE job of n_queries x N queries, rank r owns query block r with "
                         "its own engine and clock, T2 budgets allocated over every rank's candidates through "
                         "peer-memory outboxes (weak scaling: per-GPU queries fixed); independent: each rank a "
                         "whole search of its own queries (run seed + rank, weak scaling, no exchange); coupled: "
                         "ONE search, the control replicated on every rank and the model work of query block r "
                         "on rank r (single virtual clock, global T2; strong scaling)")
    ap.add_argument("--control-only", type=int, default=296,
                    help="also time N control-only searches in one batched launch (no model), 0 = off")
    ap.add_argument("--named-shapes", type=int, default=1,
                    help="also time config 5 with the Llama-3-8B-shaped policy + 1.5B-shaped PRM (1 = on)")
    return ap.parse_args()


# SPEX_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 with a gloo process
# group, so the multi-rank path (outbox exchange, reductions) runs on one GPU
ONE_GPU = os.environ.get("SPEX_BENCH_ONE_GPU") == "1"


def dist_env():
    local = 0 if ONE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), local


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks():
    try:
        return json.loads(PEAKS.read_text()), "measured"
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK_GBS, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- reference arm
def ref_lib():
    so = ROOT / "oracle" / "_ref" / "libspexref.so"
    if not so.exists():
        return None
    L = ctypes.CDLL(str(so))
    L.ref_run_timed.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    return L


def ref_runs(cfg_text: str, seeds, threads: int):
    """Independent reference runs (Executor::run, trace off) on `threads` host
    threads (ctypes releases the GIL), like run_experiment_full's OpenMP loop."""
    L = ref_lib()
    queries = [0.0] * len(seeds)
    lock = threading.Lock()
    it = iter(list(enumerate(seeds)))

    def worker():
        while True:
            with lock:
                try:
                    i, s = next(it)
                except StopIteration:
                    return
            secs = ctypes.c_double()
            tot = (ctypes.c_double * 24)()
            rc = L.ref_run_timed(cfg_text.encode(), s, None, 0, 1, ctypes.byref(secs), tot)
            if rc != 0:
                raise RuntimeError(f"reference run failed rc={rc}")
            queries[i] = tot[5]
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker) for _ in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return sum(queries), time.perf_counter() - t0


def cpu_baseline(cfg_text: str, seed: int, runs: int):
    if ref_lib() is None:
        return None
    q, secs = ref_runs(cfg_text, [seed + i for i in range(runs)], 1)
    return {"value": q / secs, "unit": "queries/s", "cores": 1, "kind": "reference",
            "sample": f"{runs} single-thread Executor::run of the same config (seeds {seed}..{seed + runs - 1}), "
                      f"{secs:.1f} s; the reference decode is a virtual clock (no model compute)"}


def run_reference(args, cfg_text, seed, rank, world):
    if rank != 0:
        return
    ncores = os.cpu_count() or 1
    metric = "ToT queries/sec"
    if ref_lib() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libspexref.so not built"}))
        return
    per_step = ncores
    for _ in range(args.warmup):
        ref_runs(cfg_text, [seed + i for i in range(per_step)], ncores)
    tq, tt = 0.0, 0.0
    for k in range(args.steps):
        q, s = ref_runs(cfg_text, [seed + 1000 * k + i for i in range(per_step)], ncores)
        tq += q
        tt += s
    v = tq / tt
    line = {"metric": metric, "value": v, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * tt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": args.config, "queries_per_search": json.loads(cfg_text)["run"]["n_queries"],
                       "searches_per_step": per_step},
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": ncores, "kind": "reference",
                             "sample": f"{per_step} concurrent Executor::run per step on {ncores} host threads"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "work_note": "the reference prices decode with a virtual clock and runs no model: this arm does the "
                         "search control only; the GPU arm's `control_only` object measures the same work"}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ ours
def main():
    args = parse()
    rank, world, local = dist_env()
    cfg_text = (ROOT / "configs" / f"{args.config}.json").read_text()
    cfg = json.loads(cfg_text)
    base_seed = cfg["run"]["seed"]
    coupled = args.sharding == "coupled"
    split = args.sharding == "split" and world > 1
    # independent: disjoint query sets per rank (weak scaling); coupled: one
    # search whose query blocks' model work is split over the ranks; split: one
    # job of n_queries x world queries, rank r owning block r (weak scaling)
    seed = base_seed if (coupled or split) else shard_seed(base_seed, rank)
    q_lo, q_hi = query_block(cfg["run"]["n_queries"], rank, world) if coupled else (0, cfg["run"]["n_queries"])
    job_text = cfg_text
    if split:
        job = json.loads(cfg_text)
        job["run"]["n_queries"] = cfg["run"]["n_queries"] * world
        job_text = json.dumps(job)
    if args.impl == "reference":
        run_reference(args, cfg_text, base_seed, rank, world)
        return

    import torch
    import paper_2605_10195_b200 as spex
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if ONE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist

    def barrier():
        torch.cuda.synchronize()
        if pg:
            pg.barrier()

    boxes, epoch, split_note = None, [0], None
    if split:
        from paper_2605_10195_b200 import _lib, shard
        try:
            boxes = shard.Outboxes(_lib.lib(), rank, world, cfg["run"]["n_queries"] * world, device=local)
        except shard.SplitUnavailable as e:  # raised on every rank alike: all run independent shards
            split, split_note = False, f"split sharding unavailable ({e}); independent shards instead"
            seed = shard_seed(base_seed, rank)
            job_text = cfg_text

    def one_search(trace: bool, flags=None):
        ex = spex.Executor(job_text, seed, flags, trace=trace, device=local)
        ex.set_model(args.policy, args.prm, weight_seed=1)
        if ONE_GPU and world > 1:
            ex.set_kv_pages(110000)  # the ranks share one GPU's HBM (tests only)
        if coupled:
            ex.set_shard(rank, world)
        if split:
            epoch[0] += 1  # the same on every rank: every rank runs the same searches
            ex.set_split(rank, world, boxes.pointers, epoch[0])
        tot = ex.run()
        tot.queries = q_hi - q_lo  # queries whose model work ran here
        d2h = 0
        if trace:
            log = ex.log_lines()  # the run's event log, copied back and serialised
            d2h = ex.stats()["log_records"] * 48
        st, ms = ex.stats(), ex.model_stats()
        ms["p50_latency_virtual_s"] = statistics.median(ex.query_finish_times())
        ex.close()
        return tot, st, ms, d2h

    for _ in range(args.warmup):
        one_search(False)
    barrier()
    peaks, peak_src = load_peaks()
    with Clocks(local) as clk:
        # device-resident value: inputs (config, weights, pools) already on the GPU
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        t0 = time.perf_counter()
        agg = {"queries": 0, "ctl_ms": 0.0, "model_ms": 0.0, "step_ms": 0.0, "streamed": 0, "attn_ms": 0.0,
               "attn_bytes": 0.0,
               "launches": 0, "flops": 0.0, "decode_rows": 0, "prm_rows": 0, "attn_launches": 0, "prm_thoughts": 0}
        for _ in range(args.steps):
            tot, st, ms, _ = one_search(False)
            agg["queries"] += tot.queries
            agg["ctl_ms"] += st["device_ms"]
            agg["model_ms"] += ms["model_ms"]
            agg["step_ms"] += ms["step_ms"]
            agg["streamed"] += ms["streamed"]
            agg["attn_ms"] += ms["attn_ms"]
            agg["attn_bytes"] += ms["attn_alg_bytes"]
            agg["attn_launches"] += ms["attn_launches"]
            agg["launches"] += 1 + ms["launches"]
            agg["flops"] += ms["policy_flops"] + ms["prm_flops"]
            agg["decode_rows"] += ms["decode_rows"]
            agg["prm_rows"] += ms["prm_rows"]
            agg["prm_thoughts"] += ms["prm_thoughts"]
        barrier()
        wall = time.perf_counter() - t0
        # device time of the step: control-kernel start -> last of (control end,
        # forward end), CUDA events; the forward streams concurrently with control
        dev_s = agg["step_ms"] / 1000.0
        # end to end through the public API (Executor: config JSON in, totals
        # back to the host), like the reference arm's Executor::run with no trace
        barrier()
        t1 = time.perf_counter()
        e2e_q = 0
        for _ in range(args.steps):
            tot, st, ms, _ = one_search(False)
            e2e_q += tot.queries
        barrier()
        e2e_wall = time.perf_counter() - t1
        # the same with the event log copied back and serialised (run_once semantics)
        barrier()
        t2 = time.perf_counter()
        tr_q, e2e_d2h = 0, 0
        for _ in range(args.steps):
            tot, st, ms, d2h = one_search(True)
            tr_q += tot.queries
            e2e_d2h += d2h
        barrier()
        tr_wall = time.perf_counter() - t2
    # the search path alone, as the reference arm runs it (virtual decode, no
    # model): independent searches in one control-kernel launch, one CTA each
    # (the device analog of the reference's OpenMP loop over repetitions)
    ctl_only = None
    if args.control_only > 0:
        n_b = args.control_only
        spex.run_batch(cfg_text, [seed + k for k in range(n_b)], device=local)  # warm-up
        t0c = time.perf_counter()
        tots_b, ms_b = spex.run_batch(cfg_text, [seed + 1000 + k for k in range(n_b)], device=local)
        wall_c = time.perf_counter() - t0c
        ctl_only = {"searches": n_b, "queries_per_s": sum(t.queries for t in tots_b) / wall_c,
                    "queries_per_s_device": sum(t.queries for t in tots_b) / (ms_b / 1000.0),
                    "wall_s": wall_c, "device_ms": ms_b,
                    "note": "device control kernel only (the reference arm's virtual-clock decode, no model): "
                            "one launch, one CTA (SM) per search; compare with --impl reference"}
    # the named model shapes (north star): config 5, Llama-3-8B-shaped policy +
    # 1.5B-shaped PRM, one warm + one timed search on this GPU
    named = None
    if args.named_shapes:
        c5 = (ROOT / "configs" / "c5_rebase_w32_q64.json").read_text()

        def c5_search():
            ex = spex.Executor(c5, json.loads(c5)["run"]["seed"] + rank, None, trace=False, device=local)
            ex.set_model("llama3_8b", "prm_1p5b", weight_seed=1)
            t = ex.run()
            m = ex.model_stats()
            m["kv"] = ex.kv_stats()
            ex.close()
            return t, m

        c5_search()
        n_tot, n_ms = c5_search()
        sec = n_ms["step_ms"] / 1000.0
        named = {"workload": "c5_rebase_w32_q64: rebase_bfs w32 d16 target32, T1+T2+T3, 64 queries",
                 "policy": "llama3_8b (32 L, d 4096, 32/8 heads x 128, FFN 14336, vocab 128256)",
                 "prm": "prm_1p5b (28 L, d 1536, 12/2 heads x 128, FFN 8960)",
                 "queries_per_s": n_tot.queries / sec, "thoughts_per_s": n_ms["prm_thoughts"] / sec,
                 "step_ms": n_ms["step_ms"], "decode_rows": n_ms["decode_rows"], "prm_rows": n_ms["prm_rows"],
                 "streamed": n_ms["streamed"],
                 "tree_kv": {"pool_pages": n_ms["kv"]["pages"], "page_tokens": n_ms["kv"]["page_tokens"],
                             "peak_live_pages": n_ms["kv"]["peak_pages"],
                             "pages_handed_out": n_ms["kv"]["allocated_pages"],
                             "distinct_pages_touched": n_ms["kv"]["fresh_pages"],
                             "bytes_per_token": 4 * (32 * 8 * 128 + 28 * 2 * 128)},
                 "k1_hbm_frac": (n_ms["attn_alg_bytes"] / (n_ms["attn_ms"] / 1000.0) / 1e9) / load_peaks()[0]["hbm_gbs"],
                 "projection_tflops": (n_ms["policy_flops"] + n_ms["prm_flops"]) / sec / 1e12,
                 "projection_tensor_frac": (n_ms["policy_flops"] + n_ms["prm_flops"]) / sec / 1e12 /
                 load_peaks()[0].get("bf16_tflops_sustained", load_peaks()[0].get("bf16_tflops", 1590.0))}
    # model mode: the PRM's scores are the rewards (awaited on device by the
    # control kernel), so the GPU sees the reward barrier; per-query device
    # wall-clock latency of SPEX (the config's flags) vs barrier-synchronous
    model_mode = None
    if world == 1:
        def mm_search(flags):
            ex = spex.Executor(cfg_text, seed, flags, trace=False, device=local)
            ex.set_model(args.policy, args.prm, weight_seed=1)
            ex.set_reward_source("prm")
            t = ex.run()
            m = ex.model_stats()
            wall_ms, wait_ms = ex.query_wall_ms()
            ex.close()
            return t, m, wall_ms, wait_ms

        model_mode = {"note": "rewards = PRM scores (K4), the control kernel waits on device for each scored "
                              "thought; device wall clock from the run start to each query_done"}
        for name, flags in (("spex", None), ("barrier_sync", "")):
            mm_search(flags)  # warm-up (its own schedule shapes)
            t_m, m_m, wall_ms, wait_ms = mm_search(flags)
            model_mode[name] = {"queries_per_s": t_m.queries / (m_m["step_ms"] / 1000.0),
                                "p50_query_latency_ms": statistics.median(wall_ms),
                                "p90_query_latency_ms": sorted(wall_ms)[int(0.9 * (len(wall_ms) - 1))],
                                "step_ms": m_m["step_ms"], "control_reward_wait_ms": wait_ms,
                                "decode_rows": m_m["decode_rows"], "prm_thoughts": m_m["prm_thoughts"],
                                "virtual_makespan": t_m.makespan}
        model_mode["p50_latency_speedup"] = (model_mode["barrier_sync"]["p50_query_latency_ms"] /
                                             model_mode["spex"]["p50_query_latency_ms"])
        model_mode["queries_per_s_speedup"] = (model_mode["spex"]["queries_per_s"] /
                                               model_mode["barrier_sync"]["queries_per_s"])
        # config 3 (rstar_dfs, T1+T2+T3, 512 queries): where the reference's
        # virtual clock shows speculation paying off (185 s vs 258 s makespan)
        c3 = (ROOT / "configs" / "c3_rstar_w4_q512.json").read_text()
        c3_seed = json.loads(c3)["run"]["seed"]
        mm3 = {"workload": "c3_rstar_w4_q512: rstar_dfs w4 d16 target10, T1+T2+T3, 512 queries"}
        for name, flags in (("spex", None), ("barrier_sync", "")):
            def c3_search():
                ex = spex.Executor(c3, c3_seed, flags, trace=False, device=local)
                ex.set_model(args.policy, args.prm, weight_seed=1)
                ex.set_reward_source("prm")
                t = ex.run()
                m = ex.model_stats()
                wall_ms, wait_ms = ex.query_wall_ms()
                ex.close()
                return t, m, wall_ms, wait_ms
            c3_search()
            t_m, m_m, wall_ms, wait_ms = c3_search()
            mm3[name] = {"queries_per_s": t_m.queries / (m_m["step_ms"] / 1000.0),
                         "p50_query_latency_ms": statistics.median(wall_ms), "step_ms": m_m["step_ms"],
                         "control_reward_wait_ms": wait_ms, "decode_rows": m_m["decode_rows"],
                         "virtual_makespan": t_m.makespan}
        mm3["p50_latency_speedup"] = mm3["barrier_sync"]["p50_query_latency_ms"] / mm3["spex"]["p50_query_latency_ms"]
        mm3["queries_per_s_speedup"] = mm3["spex"]["queries_per_s"] / mm3["barrier_sync"]["queries_per_s"]
        model_mode["c3"] = mm3
    # the same search barrier-synchronously (no T1/T2/T3: the reference's
    # baseline arm, experiment.cpp:68-70), same model work, for the metric's
    # "vs barrier-synchronous search"
    one_search(False, "")  # warm-up (its own schedule shapes)
    bs_tot, bs_st, bs_ms, _ = one_search(False, "")
    sp_makespan = tot.makespan
    red_dev = "cpu" if ONE_GPU else "cuda"
    times = torch.tensor([dev_s, wall, e2e_wall, tr_wall], dtype=torch.float64, device=red_dev)
    if pg:
        pg.all_reduce(times, op=pg.ReduceOp.MAX)
        qt = torch.tensor([float(agg["queries"]), float(e2e_q), float(tr_q)], dtype=torch.float64, device=red_dev)
        pg.all_reduce(qt)
        total_q, total_e2e_q, total_tr_q = qt.tolist()
    else:
        total_q, total_e2e_q, total_tr_q = float(agg["queries"]), float(e2e_q), float(tr_q)
    dev_s, wall, e2e_wall, tr_wall = times.tolist()
    if rank != 0:
        return
    achieved = agg["attn_bytes"] / (agg["attn_ms"] / 1000.0) / 1e9 if agg["attn_ms"] > 0 else 0.0
    traffic, traffic_alg = None, None
    if PROFILE_TRAFFIC.exists():  # committed ncu --set full capture of K1 (profiles/k1_traffic.json)
        try:
            tj = json.loads(PROFILE_TRAFFIC.read_text())
            traffic, traffic_alg = tj.get("dram_bytes_per_launch"), tj.get("alg_bytes_per_launch")
        except Exception:
            traffic = None
    clocks = clk.summary()
    # reported on rank 0 at N=1 only (the reference arm times all host cores separately)
    cpu = cpu_baseline(cfg_text, base_seed, args.cpu_sample_runs) if world == 1 else None
    line = {
        "metric": "ToT queries/sec",
        "value": total_q / dev_s,
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * dev_s / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if coupled else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (hash-seeded prompts and teacher-forced tokens, random-init weights)",
        "config": {"workload": f"{args.config}: {cfg['family']} w{cfg['policy'].get('width', 4)} "
                               f"d{cfg['policy'].get('max_depth', 16)} target{cfg['policy'].get('target_answers', 10)}, "
                               f"{'+'.join(f.upper() for f in cfg['run'].get('flags', [])) or 'no flags'}, "
                               f"{cfg['run']['n_queries']} queries/{'step' if coupled else 'GPU/step'}",
                   "policy": args.policy, "prm": args.prm,
                   "queries_per_step_per_gpu": cfg["run"]["n_queries"],
                   "l2": "inputs larger than L2 (tree KV pools of tens of GB per search)",
                   "parallelism": (f"query-block model work x{world}, search replicated (single virtual clock)"
                                   if coupled else
                                   f"query-sharded x{world}, one job, T2 budget exchange between the control "
                                   f"kernels through peer-memory outboxes" if split else
                                   f"query-sharded x{world}" + (f" ({split_note})" if split_note else ""))},
        "e2e": {"value": total_e2e_q / e2e_wall, "unit": "queries/s",
                "h2d_bytes_per_step": len(cfg_text.encode()),
                "d2h_bytes_per_step": 256 + 256 * cfg["run"]["n_queries"],
                "traced": {"value": total_tr_q / tr_wall, "unit": "queries/s",
                           "d2h_bytes_per_step": int(e2e_d2h / args.steps) + 256,
                           "note": "event log copied back and serialised to JSON lines each step"}},
        "vs_barrier_sync": {"barrier_sync_queries_per_s": bs_tot.queries / (bs_ms["step_ms"] / 1000.0),
                            "speedup": (total_q / dev_s / world) / (bs_tot.queries / (bs_ms["step_ms"] / 1000.0)),
                            "virtual_makespan_spex": sp_makespan, "virtual_makespan_barrier_sync": bs_tot.makespan,
                            "p50_search_latency_virtual_s": {"spex": ms["p50_latency_virtual_s"],
                                                             "barrier_sync": bs_ms["p50_latency_virtual_s"]},
                            "barrier_sync_decode_steps": bs_ms["decode_steps"],
                            "barrier_sync_decode_rows": bs_ms["decode_rows"],
                            "spex_decode_steps": ms["decode_steps"], "spex_decode_rows": ms["decode_rows"],
                            "note": "one GPU, same config/seed/model, flags '' vs the config's flags; "
                                    "device step time of one warm search each"},
        "work_note": "value/e2e include the real policy decode and PRM scoring of every scheduled row, which the "
                     "reference only prices (virtual clock, no model); `control_only` is the like-for-like "
                     "comparison with the reference arm",
        "thoughts_per_s": agg["prm_thoughts"] / dev_s,
        "named_model_shapes": named,
        "model_mode": model_mode,
        "control_only": ctl_only,
        "gpu_launches": int(agg["launches"]),
        "roofline": {"bound": "hbm", "kernel": "K1 tree_attn_bulk_kernel (policy decode rows, bulk-copy pipeline)",
                     "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "traffic_alg_bytes_same_launches": traffic_alg,
                     "alg_bytes_per_launch": agg["attn_bytes"] / max(1, agg["attn_launches"]),
                     "peak_source": peak_src,
                     "k1_share_of_step": (agg["attn_ms"] / 1000.0) / dev_s if dev_s > 0 else None},
        "cpu_baseline": cpu,
        "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "breakdown": {"streamed_steps": agg["streamed"],
                      "control_ms_per_step": agg["ctl_ms"] / args.steps,
                      "model_ms_per_step": agg["model_ms"] / args.steps,
                      "k1_ms_per_step": agg["attn_ms"] / args.steps,
                      "decode_rows_per_step": agg["decode_rows"] / args.steps,
                      "prm_rows_per_step": agg["prm_rows"] / args.steps,
                      "projection_tflops": agg["flops"] / (agg["model_ms"] / 1000.0) / 1e12
                      if agg["model_ms"] > 0 else None,
                      "wall_s_per_step": wall / args.steps},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
