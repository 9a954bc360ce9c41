#!/usr/bin/env python
"""Benchmark of the B200 MESSI exact 1-NN hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode ed|dtw]

One STEP = a batch of Q queries (default 100, the paper's query-set size) answered
one after the other (the paper's sequential model) by the whole hot path
(A3-A10: prologue/approximate search, LB scan + compaction, refine, exact re-rank, and for
N > 1 the cross-GPU merge) over the workload's collection, inputs resident in HBM.  The
index build (A1 summarise + A2 key sort) runs once per collection and is reported in
"build".  N = 1 workload: config 3 (100M x 256, ED) -- the collection the metric is quoted
on -- fits one B200; for N > 1 the same collection is row-sharded (strong scaling).  DTW
(config 4: 10M x 256, reach 25) is reported in "dtw" (or as the headline with --mode dtw).

--impl reference times the CPU oracle (the reference arm for this tier) on a bounded row
sample of the same workload, on the host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exact 1-NN queries/sec (ED & DTW, 100M×256 fp32) at 1/2/4/8 B200; % HBM roofline"
PAPER_QPS = 20.0  # ~50 ms per exact ED 1-NN query on 100M x 256, 2x Xeon E5-2650 v4

CONFIGS = {
    "c1": dict(N=100_000, n=256, Q=10, reach=None, name="C1 ED exact 1-NN tiny: 100,000 x 256 random walks"),
    "c2": dict(N=10_000_000, n=256, Q=100, reach=None, name="C2 ED exact 1-NN: 10,000,000 x 256 random walks"),
    "c3": dict(N=100_000_000, n=256, Q=100, reach=None,
               name="C3 ED exact 1-NN: 100,000,000 x 256 z-normalised random walks (seed 0), 100 random-walk "
                    "queries (seed 1), iSAX w=16 card 256, row-sharded over the GPUs"),
    "c4": dict(N=10_000_000, n=256, Q=100, reach=25,
               name="C4 DTW exact 1-NN: 10,000,000 x 256 random walks, Sakoe-Chiba reach 25 (10%), 100 queries"),
    "c5": dict(N=100_000_000, n=128, Q=1000, reach=None, noisy=True,
               name="C5 ED exact 1-NN tight pruning: 100,000,000 x 128, 1,000 noisy dataset queries (sigma 0.1)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="ed", choices=["ed", "dtw"])
    ap.add_argument("--config", default=None, help="c1..c5 (default: c3 for ed, c4 for dtw)")
    ap.add_argument("--rows", type=int, default=None, help="override the collection size")
    ap.add_argument("--queries", type=int, default=None, help="override queries per step")
    ap.add_argument("--no-dtw", action="store_true", help="skip the secondary DTW measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle timing")
    ap.add_argument("--cpu-queries", type=int, default=32, help="queries of the oracle timing sample")
    ap.add_argument("--steady", type=int, default=500000,
                    help="DTW: candidates of the steady-state refine measurement (0: skip)")
    ap.add_argument("--window", type=int, default=0, help="approximate-search window (0: library default 2000)")
    ap.add_argument("--knn", type=int, default=10, help="ED: also time exact k-NN with this k (<= 1: skip)")
    ap.add_argument("--latency", type=int, default=20,
                    help="1 GPU: also time this many single-query calls (latency mode, p50/p99; 0: skip)")
    ap.add_argument("--no-share-bsf", action="store_true",
                    help="N > 1: do not link the shards (no best-so-far sharing over peer memory)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: host-side merge; lets several ranks share one GPU)")
    ap.add_argument("--repeats", type=int, default=10,
                    help="repeat the timed K steps this many times for mean / range (P:2022-2023)")
    ap.add_argument("--dump-results", default=None,
                    help="rank 0 writes the merged (d2, gid) of the last timed step to this .npz (tests)")
    return ap.parse_args()


# ------------------------------------------------------------------------ dist plumbing
def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch
        import torch.distributed as dist
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator's init lines (nranks) on stderr
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """`bench.py --gpus N` without a launcher: start N ranks of this script (one process per
    GPU, RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* set as torchrun would), wait for them, and
    exit with the first failure.  Rank 0 prints the JSON line."""
    import subprocess
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE=str(args.gpus),
               LOCAL_WORLD_SIZE=str(args.gpus))
    procs = [subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                              env=dict(env, RANK=str(r), LOCAL_RANK=str(r))) for r in range(args.gpus)]
    rc = 0
    while procs:
        for p in list(procs):
            code = p.poll()
            if code is None:
                continue
            procs.remove(p)
            if code != 0 and rc == 0:
                rc = code
                for q in procs:  # a failed rank would leave the others waiting in a collective
                    q.terminate()
        time.sleep(0.2)
    sys.exit(rc)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent NVML sampling of SM clock and throttle reasons while running."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# --------------------------------------------------------------------------- our arm
def gen_collection(cfg, rank, world, dev):
    import torch
    import datagen
    from paper_2110_07519_b200.dist import shard_range
    b, e = shard_range(cfg["N"], world, rank)
    X = torch.empty((e - b, cfg["n"]), dtype=torch.float32, device=dev)
    datagen.walks_cuda(X, b, seed=datagen.DATA_SEED)
    Q = torch.empty((cfg["Q"], cfg["n"]), dtype=torch.float32, device=dev)
    if cfg.get("noisy"):
        datagen.noisy_queries_cuda(Q, cfg["N"], sigma=0.1)
    else:
        datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
    torch.cuda.synchronize()
    return X, Q, b


def run_arm(cfg, args, world, rank, dev, stream, time_steps, warmup, repeats=1):
    """Build + time `time_steps` steps of cfg's queries.  Returns a dict of measurements."""
    import torch
    from paper_2110_07519_b200 import messi as M
    from paper_2110_07519_b200.dist import merge_results

    X, Q, row_begin = gen_collection(cfg, rank, world, dev)
    reach = cfg["reach"]
    with torch.cuda.stream(stream):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        idx = M.Index(X, row_begin=row_begin, stream=stream, window=args.window)
        t1.record(stream)
        if world > 1 and not args.no_share_bsf:
            from paper_2110_07519_b200.dist import link_shards
            link_shards(idx)  # shards share each query's best-so-far over peer memory (NVLink)
        torch.cuda.synchronize()
        build_ms = t0.elapsed_time(t1)
        build_phases = M.messi_build_times(idx.handle)
        nq = Q.shape[0]
        res = M.result_buffer(nq, dev)
        stats = M.stats_buffer(nq, dev)
        merged = {}

        def step():
            idx.query_batch(Q, reach, res, stats)
            if world > 1:
                dist_, gid, d2 = M.decode_results_device(res)
                merged["d2"], merged["gid"] = merge_results(d2, gid)

        # NVML comes up BEFORE the warm-up (its first init takes tens of ms of host time, during
        # which the GPU would sit idle between the warm-up and the timed steps: the first repeat
        # then ran 2-3 % below the others)
        samplers = [ClockSampler(dev.index or 0) for _ in range(max(1, repeats))]
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        rep_ms = []
        launches = 0
        clk_all = []
        for rpt in range(max(1, repeats)):
            barrier(world)
            torch.cuda.synchronize()
            launches0 = idx.launches()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            with samplers[rpt] as clk:
                ev0.record(stream)
                for _ in range(time_steps):
                    step()
                ev1.record(stream)
                torch.cuda.synchronize()
            barrier(world)
            torch.cuda.synchronize()
            rep_ms.append(ev0.elapsed_time(ev1))
            clk_all.append(clk)
            if rpt == 0:
                launches = idx.launches() - launches0
        ms = rep_ms[0]
        if world == 1:
            _, gid, d2 = M.decode_results(res)
            merged = {"d2": d2, "gid": gid}
        last = {k: v.cpu() for k, v in merged.items()}
        st = M.decode_stats(stats)
        # per-kernel breakdown: the same steps again with a CUDA event pair around every launch
        # on its own stream (kept out of the timed region above: the events cost time).  The
        # per-query (DTW) path runs this pass SERIALLY -- every stage on the index stream, no
        # overlap -- so each kernel's time is its own and the times add up to the pass.
        M.messi_profile_enable(idx.handle, True, serial=reach is not None)
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(time_steps):
            step()
        p1.record(stream)
        torch.cuda.synchronize()
        prof_ms = p0.elapsed_time(p1)
        prof = {k: M.messi_profile_read(idx.handle, k) for k in ("seed", "scan", "refine", "lbk", "resolve")}
        M.messi_profile_enable(idx.handle, False)

        # e2e: the same steps through the public API with HOST buffers: pinned host queries
        # -> H2D, the batch call, D2H of the results (and the merge for N > 1), every step.
        qh = Q.cpu().pin_memory()
        rh = torch.empty(res.numel(), dtype=torch.uint8).pin_memory()
        qd = torch.empty_like(Q)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)

        def e2e_step():
            qd.copy_(qh, non_blocking=True)
            idx.query_batch(qd, reach, res, None)
            if world > 1:
                dist_, gid, d2 = M.decode_results_device(res)
                merge_results(d2, gid)
            rh.copy_(res, non_blocking=True)

        for _ in range(warmup):  # untimed: the pinned allocations above left the GPU idle
            e2e_step()
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(time_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        e2e_ms = e0.elapsed_time(e1)
        # exact k-NN (f2) on the same index and queries: k = args.knn results per query
        knn = None
        if reach is None and args.knn > 1:
            from paper_2110_07519_b200.dist import merge_knn
            kres = M.result_buffer(nq * args.knn, dev)

            def kstep():
                idx.query_batch_knn(Q, args.knn, kres)
                if world > 1:
                    _, kid, kd2 = M.decode_results_device(kres)
                    merge_knn(kd2.view(nq, args.knn), kid.view(nq, args.knn))

            for _ in range(max(1, warmup)):
                kstep()
            torch.cuda.synchronize()
            barrier(world)
            k0 = torch.cuda.Event(enable_timing=True)
            k1 = torch.cuda.Event(enable_timing=True)
            k0.record(stream)
            for _ in range(time_steps):
                kstep()
            k1.record(stream)
            torch.cuda.synchronize()
            barrier(world)
            knn = k0.elapsed_time(k1)
        # latency mode (SURVEY 8(d) protocol, the paper's one-query-at-a-time model P:2024-2026):
        # the synchronous single-query call, query from pinned host memory to result in host
        # memory, CUDA events on the index stream around each call
        lat = []
        if world == 1 and args.latency > 0:
            qh1 = Q[: min(nq, args.latency)].cpu().pin_memory()
            for i in range(min(3, qh1.shape[0])):  # warm-up
                idx.query_ed(qh1[i]) if reach is None else idx.query_dtw(qh1[i], reach)
            for i in range(qh1.shape[0]):
                l0 = torch.cuda.Event(enable_timing=True)
                l1 = torch.cuda.Event(enable_timing=True)
                l0.record(stream)
                idx.query_ed(qh1[i]) if reach is None else idx.query_dtw(qh1[i], reach)
                l1.record(stream)
                torch.cuda.synchronize()
                lat.append(l0.elapsed_time(l1))
        # DTW refine kernel at steady state: the query path's refine kernel over a long list of
        # candidates in its inspection mode (frozen: every candidate runs all n rows, no abandon)
        # -- its cell rate without the per-query tail of a short list; CUDA events around the
        # refine launch (messi_debug_dtw_stages, profiling on)
        steady = None
        if world == 1 and reach is not None and args.steady > 0:
            ids = torch.arange(min(args.steady, X.shape[0]), dtype=torch.int32, device=dev)
            M.messi_debug_dtw_stages(idx.handle, Q[0].contiguous(), reach, ids)  # warm-up
            torch.cuda.synchronize()
            M.messi_profile_enable(idx.handle, True)
            M.messi_debug_dtw_stages(idx.handle, Q[0].contiguous(), reach, ids)
            torch.cuda.synchronize()
            sms, _ = M.messi_profile_read(idx.handle, "refine")
            M.messi_profile_enable(idx.handle, False)
            n_, r_ = cfg["n"], min(reach, cfg["n"] - 1)
            cells = ids.numel() * (n_ * (2 * r_ + 1) - r_ * (r_ + 1))
            steady = {"candidates": ids.numel(), "cells": cells, "ms": sms}
    build_phases = {**build_phases, "renv": M.messi_build_times(idx.handle)["renv"]}  # DTW: after its first query
    out = dict(ms=ms, rep_ms=rep_ms, build_ms=build_ms, build_phases=build_phases, launches=launches, prof=prof,
               prof_ms=prof_ms, stats=st, clocks=clk_all[0].summary(), e2e_ms=e2e_ms, knn_ms=knn, nq=nq,
               N_local=X.shape[0], n=cfg["n"], reach=reach, h2d=qh.numel() * 4, d2h=rh.numel(), latency_ms=lat,
               last=last, steady=steady)
    idx.close()
    del X, Q
    torch.cuda.empty_cache()
    return out


def tc_compare(idx, Q, dev, stream, reps=5):
    """The tensor-core batched path (SURVEY 8(f) f4 (i)+(ii)) against the LUT batch path on one
    index and query set: q/s of each, the TC kernel's own time, its rows8 stream rate (of the
    measured HBM peak) and int8 tensor rate (of 2 x the measured bf16 peak: the guide's nominal
    int8 / bf16 ratio), and whether both paths return the same answers."""
    import torch
    from paper_2110_07519_b200 import messi as M
    nq = Q.shape[0]
    r1, r2, st = M.result_buffer(nq, dev), M.result_buffer(nq, dev), M.stats_buffer(nq, dev)
    out = {"queries": nq}
    with torch.cuda.stream(stream):
        for name, fn in (("lut", lambda: idx.query_batch(Q, None, r1)), ("tc", lambda: idx.query_batch_tc(Q, r2, st))):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out[name] = {"ms": ms, "qps": nq / (ms / 1e3)}
        M.messi_profile_enable(idx.handle, True)
        idx.query_batch_tc(Q, r2, st)
        kms = M.messi_profile_read(idx.handle, "scan")[0]
        M.messi_profile_enable(idx.handle, False)
        torch.cuda.synchronize()
    a, b = M.decode_results(r1), M.decode_results(r2)
    sts = M.decode_stats(st)
    pk = peaks()
    N, n = idx.count, idx.n
    gbs = N * (n + 16) / (kms / 1e3) / 1e9  # rows8 + the 16 B row term per row
    tops = 2.0 * N * n * nq / (kms / 1e3) / 1e12
    int8_peak = 2.0 * pk.get("bf16_tflops", 1590.0)
    out["tc"].update({"kernel": "k_ed_tc (TMA ring of int8 rows -> tcgen05.mma kind::i8 -> TMEM -> epilogue test)",
                      "kernel_ms": kms, "hbm_gbs": gbs, "hbm_frac": gbs / pk.get("hbm_gbs", 6650.0),
                      "int8_tops": tops, "int8_peak_tops": int8_peak, "tensor_frac": tops / int8_peak,
                      "candidates_mean": sum(x["candidates"] for x in sts) / nq,
                      "exact_mean": sum(x["exact"] for x in sts) / nq,
                      "same_answers_as_lut": bool(torch.equal(a[1], b[1]) and torch.equal(a[2], b[2]))})
    return out


def build_split(args, dev, stream):
    """Index build of config 2 (10M x 256) on this GPU, phase by phase (device events inside
    messi_build): summarise (A1: 4n B read + 24 B written per series, the HBM-bound pass SURVEY
    8(d) prices at 1,104 B/series), key sort, sorted layout, quantised rows."""
    import torch
    import datagen
    from paper_2110_07519_b200 import messi as M
    c2 = CONFIGS["c2"]
    X, _, _ = gen_collection(dict(c2, Q=1), 0, 1, dev)
    with torch.cuda.stream(stream):
        idx = M.Index(X, stream=stream, window=args.window)  # warm-up build (allocations, first launches)
        idx.close()
        torch.cuda.synchronize()
        idx = M.Index(X, stream=stream, window=args.window)
        torch.cuda.synchronize()
        ph = M.messi_build_times(idx.handle)
    tc = {}
    for nq in (100, 256):  # C2's query set, and a full tensor-core pass
        Q = torch.empty((nq, c2["n"]), dtype=torch.float32, device=dev)
        datagen.walks_cuda(Q, 0, seed=datagen.QUERY_SEED)
        torch.cuda.synchronize()
        tc[f"q{nq}"] = tc_compare(idx, Q, dev, stream)
    idx.close()
    del X
    torch.cuda.empty_cache()
    N, n = c2["N"], c2["n"]
    pk = peaks().get("hbm_gbs", 6650.0)
    summ_bytes = N * (4 * n + 28)
    return {"workload": c2["name"], "phases_ms": ph, "total_ms": sum(ph.values()),
            "series_per_s": N / (sum(ph.values()) / 1e3),
            "summarise": {"series_per_s": N / (ph["summarise"] / 1e3),
                          "achieved_gbs": summ_bytes / (ph["summarise"] / 1e3) / 1e9,
                          "frac": summ_bytes / (ph["summarise"] / 1e3) / 1e9 / pk,
                          "algorithmic_bytes": summ_bytes,
                          "what": "per series: 4n B of rows read; 16 B of symbols, 8 B of key, 4 B of row id written"},
            "tc_vs_lut": tc}


# DTW band DP roofline: a cell costs one FADD + one FFMA on the FMA pipe (plus
# an FMNMX3 on the ALU pipe); the FMA pipe retires one warp instruction per 2 cycles per SM
# sub-partition, so the fp32 cell peak is 148 SMs x 4 SMSPs x 32 lanes / (2 x 2 cycles) x clock.
def dtw_cell_peak(sm_mhz=1965.0, sms=148):
    # >= 2 issue slots per cell (FMNMX3 + paired FADD2/FFMA2), 1 warp instruction / cycle / SMSP
    return sms * 4 * 32 / 2.0 * sm_mhz * 1e6


def steady_refine(run):
    """The refine kernel's cell rate on a long frozen candidate list (run["steady"])."""
    sd = run.get("steady")
    if not sd or sd["ms"] <= 0:
        return None
    peak = dtw_cell_peak(run["clocks"].get("sm_max_mhz", 1965.0) or 1965.0)
    rate = sd["cells"] / (sd["ms"] / 1e3)
    return {"achieved": rate, "peak": peak, "unit": "cells/s", "frac": rate / peak,
            "candidates": sd["candidates"], "ms": sd["ms"],
            "what": "the same refine kernel over the first %d rows as candidates in its inspection mode "
                    "(frozen: every candidate runs all n rows), CUDA events around its launch: the kernel's "
                    "rate without the per-query tail of a short candidate list" % sd["candidates"]}


def dtw_roofline(run, steps):
    """Roofline of the DTW refine: valid band cells (counted by the kernels, SURVEY 8(d):
    n(2r+1) - r(r+1) per completed candidate, the rows done for an abandoned one) over the
    refine kernels' time in the SERIAL profiling pass (every stage alone on the stream, so
    the refine time is its own and <= that pass's step time)."""
    st = run["stats"]
    cells = sum(s["dtw_cells"] for s in st) * steps
    ms, nl = run["prof"]["refine"]
    if ms <= 0:
        return None
    achieved = cells / (ms / 1e3)
    peak = dtw_cell_peak(run["clocks"].get("sm_max_mhz", 1965.0) or 1965.0)
    lbk_ms, _ = run["prof"]["lbk"]
    # strip refine reaches (r >= 7): the reverse envelope-PAA filter reads every scan candidate's
    # entry (8 B) and envelope symbols (32 B) and writes its survivors (8 B, stats
    # "rev_paa_pass"); the forward filter reads those survivors' entries (8 B), quantised rows
    # (n bytes) and scale / error (8 B); the reverse bound (stats "exact": its evaluations)
    # writes and reads a 16 B queue entry, reads the row again and its id (4 B); every survivor
    # is a 16 B list2 entry.  Register-band reaches: raw rows (4n bytes) of every candidate
    n = run["n"]
    strip = (run.get("reach") or 0) >= 7
    renv = strip and not os.environ.get("MESSI_NO_RENV")
    per_cand = n + 16 if strip else 4 * n + 8
    lbk_bytes = sum((40 * s["candidates"] + (8 + per_cand) * s["rev_paa_pass"] if renv else per_cand * s["candidates"])
                    + (n + 36) * s["exact"] + 16 * s["lbk_pass"] for s in st) * steps
    return {"bound": "alu", "kernel": "k_refine_dtw_strip<8,REM> (fp32 banded DTW, one thread per candidate; "
                                      "k_refine_dtw<R> at R = 2, 5)",
            "achieved": achieved, "peak": peak, "unit": "cells/s", "frac": achieved / peak,
            "cells_per_step": cells / steps, "refine_ms_per_step": ms / steps,
            "serial_pass_ms_per_step": run["prof_ms"] / steps,
            "peak_source": "derived (DESIGN.md 6): issue limit 1 warp-instr / cycle / SMSP at >= 2 instr per cell "
                           "(FMNMX3 + paired FADD2/FFMA2), 148 SMs x 4 SMSP, max SM clock",
            "time": "CUDA events around the refine launches in a serial pass of the same steps (no stage overlap)",
            "steady_state": steady_refine(run),
            "lbk_filter": {"bound": "hbm", "kernels": "k_rev_paa_filter (reverse envelope-PAA bound over the scan's "
                                                      "candidates) + k_lbk_filter_q8b (forward LB_Keogh, bulk-copy "
                                                      "rows) + k_lbk_rev_q8 (reverse LB_Keogh over the forward survivors)",
                           "achieved_gbs": lbk_bytes / (lbk_ms / 1e3) / 1e9 if lbk_ms > 0 else None,
                           "frac": lbk_bytes / (lbk_ms / 1e3) / 1e9 / peaks().get("hbm_gbs", 6650.0)
                           if lbk_ms > 0 else None,
                           "ms_per_step": lbk_ms / steps, "bytes_per_query": lbk_bytes / steps / len(st)}}


def arm_config(cfg, args, world, nq):
    """The workload description both arms print (same keys, same values)."""
    nl = cfg["N"] // world
    return {"workload": cfg["name"], "mode": args.mode, "rows": cfg["N"], "length": cfg["n"],
            "queries_per_step": nq, "reach": cfg["reach"], "parallelism": f"row-shard x{world}",
            "merge": "per step: one all_gather of (d2, gid) x queries per rank, lexicographic min" if world > 1
            else "single shard",
            "l2": "inputs larger than L2: %.2f GB of coarse iSAX tiles + %.2f GB of 8-bit words + %.2f GB of "
                  "quantised rows per GPU; each query streams the tiles its box filter keeps (distinct per query)"
                  % (8 * nl / 1e9, 16 * nl / 1e9, cfg["n"] * nl / 1e9),
            "query_model": "throughput: one batch call per step, all %d queries of the step in flight "
                           "(every query answered exactly and independently); latency mode (the paper's "
                           "one query at a time, P:2024-2026) is reported in \"latency\"" % nq}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _sample_rows(cfg, rows, dev):
    """The first `rows` rows of the workload's collection (device generator, copied back)."""
    import datagen
    if dev is not None:
        import torch
        X = torch.empty((rows, cfg["n"]), dtype=torch.float32, device=dev)
        datagen.walks_cuda(X, 0, seed=datagen.DATA_SEED)
        Xh = X.cpu().numpy()
        del X
        return Xh
    return datagen.walks_cpu(0, rows, cfg["n"])


def _oracle_time(cfg, Xh, Qh, threads):
    import oracle
    t = time.perf_counter()
    oracle.nn("ed" if cfg["reach"] is None else "dtw", Xh, Qh, r=cfg["reach"] or 0, threads=threads,
              chunk=max(1, Xh.shape[0] // (4 * threads)))
    return time.perf_counter() - t


def oracle_sample_size(cfg):
    """Rows of the oracle's bounded sample (the same for cpu_baseline and the reference arm):
    4M rows for ED (about 25 core-seconds for 32 queries on 16 host threads), 20K for DTW (each
    DTW row costs n(2r+1) - r(r+1) = 12,406 fp64 cells at C4)."""
    return min(cfg["N"], 4_000_000 if cfg["reach"] is None else 20_000)


def cpu_baseline(cfg, args, dev, kind):
    """The oracle, as it stands, timed on this host's cores over a bounded row sample of the
    workload (rows copied back from the device generator), scaled to the full collection;
    plus its single-core time on C1 and on a 1M-row subset of C2."""
    import datagen
    rows = oracle_sample_size(cfg)
    Xh = _sample_rows(cfg, rows, dev)
    nq = args.cpu_queries if cfg["reach"] is None else 2
    Qh = datagen.walks_cpu(0, nq, cfg["n"], seed=datagen.QUERY_SEED)
    cores = len(os.sched_getaffinity(0))
    dt = _oracle_time(cfg, Xh, Qh, cores)
    qps = nq / (dt * cfg["N"] / rows)
    del Xh
    single = {}
    c1 = CONFIGS["c1"]
    X1 = _sample_rows(c1, c1["N"], dev)
    Q1 = datagen.walks_cpu(0, c1["Q"], c1["n"], seed=datagen.QUERY_SEED)
    single["c1_s"] = _oracle_time(c1, X1, Q1, 1)
    single["c1_what"] = "C1 ED, all 10 queries over 100,000 x 256, one core"
    del X1
    c2 = CONFIGS["c2"]
    X2 = _sample_rows(c2, 1_000_000, dev)
    Q2 = datagen.walks_cpu(0, 4, c2["n"], seed=datagen.QUERY_SEED)
    t2 = _oracle_time(c2, X2, Q2, 1)
    single["c2_1m_s_per_query"] = t2 / 4
    single["c2_1m_what"] = "C2 ED, 4 queries over the first 1,000,000 rows, one core; seconds per query"
    return {"value": qps, "unit": "queries/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{nq} queries x first {rows:,} of {cfg['N']:,} rows in {dt:.2f} s wall "
                      f"({dt * cores:.0f} core-seconds), linearly scaled to the full collection; plain fp64 "
                      f"brute force ({kind}), one serial call per row chunk on {cores} threads",
            "seconds": dt, "core_seconds": dt * cores, "single_core": single,
            "paper_context": "MESSI (CPU, 2x Xeon E5-2650 v4, 24 cores / 48 threads): ~50 ms per exact ED query "
                             "on 100M x 256 (~20 q/s, P:58, P:137, P:2881); DTW 679.3 ms RD time per query "
                             "(P:2718)"}


def ours(args):
    import torch
    if os.environ.get("MESSI_LIB") and os.environ.get("MESSI_AB") != "1":
        raise SystemExit("bench.py: MESSI_LIB is set; the bench only times the in-tree libmessi.so "
                         "(A/B experiments set MESSI_AB=1 too, and the line then names the library)")
    world, rank, local = dist_init(args)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    cname = args.config or ("c3" if args.mode == "ed" else "c4")
    cfg = dict(CONFIGS[cname])
    if args.rows:
        cfg["N"] = args.rows
    if args.queries:
        cfg["Q"] = args.queries
    if args.mode == "dtw" and cfg["reach"] is None:
        cfg["reach"] = 25
    pk = peaks()
    main = run_arm(cfg, args, world, rank, dev, stream, args.steps, args.warmup, repeats=args.repeats)
    ms = max_over_ranks(main["ms"], world)
    rep = [max_over_ranks(x, world) for x in main["rep_ms"]]
    e2e_ms = max_over_ranks(main["e2e_ms"], world)
    scan_ms, scan_n = main["prof"]["scan"]
    scan_ms = max_over_ranks(scan_ms, world)
    K, nq = args.steps, main["nq"]
    value = K * nq / (ms / 1e3)
    # roofline of the dominant kernel, k_scan_refine_ed (one launch per step for ED: the whole
    # batch).  Algorithmic bytes per launch = sum over the batch's queries of
    # 4 KB per tile scanned + 8 B per listed tile (the list entry) + 16 B per coarse survivor
    # (its 8-bit word) + n + 8 B per refined candidate (quantised row + scale / bound) + 4n B
    # per exact fp32 distance; achieved = those bytes over the kernel's own CUDA-event time.
    st = main["stats"]
    mean = lambda k: sum(s[k] for s in st) / len(st)  # noqa: E731
    tot = lambda k: sum(s[k] for s in st)  # noqa: E731
    n_ = main["n"]
    ntiles = (main["N_local"] + 511) // 512
    if cfg["reach"] is None:
        kern = "k_scan_refine_ed (fused box re-check + iSAX LB scan + quantised/fp32/fp64 refine, whole batch)"
        launch_bytes = (4096 * tot("tiles_scanned") + 8 * tot("tiles_listed") + 16 * tot("coarse")
                        + (n_ + 8) * tot("refined") + 4 * n_ * tot("exact"))
    else:
        kern = "k_scan (iSAX envelope LB scan of the box-filtered tiles, per query)"
        launch_bytes = 4096 * mean("tiles_scanned") + 16 * mean("coarse") + 8 * mean("candidates")
    achieved = launch_bytes * scan_n / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None
    peak = pk.get("hbm_gbs", 6650.0)
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tr.get(f"{cname}_{args.mode}_bytes_per_launch")
    except Exception:
        pass
    # whole-query algorithmic bytes per GPU: tile boxes (filter) + surviving tiles + list
    # entries + refine bytes + the approximate-search window rows
    per_query_bytes = (32 * ntiles + 4096 * mean("tiles_scanned") + 8 * mean("tiles_listed") + 16 * mean("coarse")
                       + (n_ + 8) * mean("refined") + 4 * n_ * mean("exact") + 4 * n_ * min(2000, main["N_local"]))
    steps_total = {k: max_over_ranks(v[0], world) for k, v in main["prof"].items()}
    lat_qps = None
    if main.get("latency_ms"):
        lat_qps = 1e3 * len(main["latency_ms"]) / sum(main["latency_ms"])
    paper_cmp = args.mode == "ed" and cname == "c3" and not args.rows
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
        # like for like with the paper's sequential queries (~20 q/s, P:58 / P:137 / P:2881): the
        # latency-mode rate (one synchronous query at a time), not the batched throughput
        "vs_baseline": (lat_qps / PAPER_QPS) if (paper_cmp and lat_qps) else None,
        "vs_baseline_basis": "latency-mode q/s (one synchronous query at a time, host in / host out) / the "
                             "paper's ~20 q/s (~50 ms per query, 100M x 256, 2x Xeon E5-2650 v4); the batched "
                             "throughput `value` / 20 is %s" % (f"{value / PAPER_QPS:.0f}" if paper_cmp else "n/a"),
        "dtype": "f32", "data": "synthetic (seeded device Philox random walks, z-normalised)",
        "config": arm_config(cfg, args, world, nq),
        "roofline": {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst; of measured)" if "hbm_gbs" in pk
                     else "fallback 6650 GB/s (of fallback)",
                     "algorithmic_bytes_per_launch": launch_bytes, "launches": scan_n,
                     "share_of_step": scan_ms / main["prof_ms"] if main["prof_ms"] else None,
                     "bytes_formula": "4096 B per tile scanned + 8 B per listed tile + 16 B per coarse survivor + "
                                      "(n + 8) B per fine survivor + 4n B per exact fp32 distance",
                     "timing": "CUDA events around every launch of the kernel on its stream, in a second "
                               "pass of the same steps (profiling events kept out of the timed region)"},
        "query_roofline": {"bytes_per_query_per_gpu": per_query_bytes,
                           "qps_at_peak": peak * 1e9 / per_query_bytes,
                           "frac": value / (peak * 1e9 / per_query_bytes)},
        "kernel_ms_per_step": {k: v / K for k, v in steps_total.items()},
        "repeats": {"n": len(rep), "qps": [K * nq / (x / 1e3) for x in rep],
                    "mean": statistics.fmean(K * nq / (x / 1e3) for x in rep),
                    "min": min(K * nq / (x / 1e3) for x in rep), "max": max(K * nq / (x / 1e3) for x in rep),
                    "what": "the timed K steps repeated back to back (the paper averages 10 runs, P:2022-2023); "
                            "value = the first"},
        "e2e": {"value": K * nq / (e2e_ms / 1e3), "unit": "queries/s", "h2d_bytes_per_step": main["h2d"],
                "d2h_bytes_per_step": main["d2h"]},
        "gpu_launches": main["launches"],
        "lib": os.environ.get("MESSI_LIB") or "paper_2110_07519_b200/libmessi.so",
        "clocks": main["clocks"],
        "build": {"ms": main["build_ms"], "rows_per_s": main["N_local"] / (main["build_ms"] / 1e3),
                  "phases_ms": main["build_phases"],
                  "what": "messi_build per GPU: breakpoints + summarise (PAA, iSAX, key) + CUB key sort + sorted "
                          "layout + quantised rows"},
        "stats_mean": {k: mean(k) for k in ("lb_computed", "tiles_scanned", "candidates", "rev_paa_pass", "lbk_pass", "refined",
                                             "abandoned", "near_best", "dtw_cells", "exact", "tiles_listed", "coarse",
                                             "seed_d2", "bsf_d2")},
    }

    def dist_of(stl):
        def q(vals, p):
            v = sorted(vals)
            return v[min(len(v) - 1, int(p * len(v)))]
        c = [x["candidates"] for x in stl]
        r = [x["refined"] for x in stl]
        ratio = [x["seed_d2"] / x["bsf_d2"] for x in stl if x["bsf_d2"] > 0]
        return {"candidates": {"mean": statistics.fmean(c), "median": statistics.median(c), "p90": q(c, 0.9)},
                "refined": {"mean": statistics.fmean(r), "median": statistics.median(r), "p90": q(r, 0.9)},
                "bsf0_over_final": {"median": statistics.median(ratio) if ratio else None,
                                    "p90": q(ratio, 0.9) if ratio else None},
                "near_best_mean": statistics.fmean(x["near_best"] for x in stl)}

    line["stats_dist"] = dist_of(main["stats"])
    if main.get("latency_ms"):
        lt = sorted(main["latency_ms"])
        line["latency"] = {"queries": len(lt), "p50_ms": lt[len(lt) // 2], "p99_ms": lt[min(len(lt) - 1, int(0.99 * len(lt)))],
                           "mean_ms": sum(lt) / len(lt), "qps": lat_qps,
                           "what": "synchronous single-query calls (host query in, host result out), CUDA events"}
    if main.get("knn_ms"):
        kms = max_over_ranks(main["knn_ms"], world)
        line["knn"] = {"k": args.knn, "value": K * nq / (kms / 1e3), "unit": "queries/s", "ms_per_step": kms / K,
                       "what": "exact k-NN (ED) of the same queries on the same index, k results per query"}
    if args.mode == "dtw":
        line["roofline"] = dtw_roofline(main, K)
    if args.mode == "ed" and not args.no_dtw:
        c4 = dict(CONFIGS["c4"])
        k4 = max(1, min(2, K))
        d = run_arm(c4, args, world, rank, dev, stream, k4, 1)
        dms = max_over_ranks(d["ms"], world)
        dst = d["stats"]
        dm = lambda k: sum(s[k] for s in dst) / len(dst)  # noqa: E731
        line["dtw"] = {"value": k4 * d["nq"] / (dms / 1e3), "unit": "queries/s", "workload": c4["name"],
                       "steps": k4, "ms_per_step": dms / k4,
                       "kernel_ms_per_step_serial": {k: v[0] / k4 for k, v in d["prof"].items()},
                       "serial_pass_ms_per_step": d["prof_ms"] / k4,
                       "stats_mean": {**{k: dm(k) for k in ("lb_computed", "tiles_scanned", "candidates",
                                                            "rev_paa_pass", "lbk_pass", "refined", "abandoned",
                                                            "near_best", "dtw_cells", "coarse", "seed_d2", "bsf_d2")},
                                      "reverse_evaluated": dm("exact")},
                       "gpu_launches": d["launches"], "roofline": dtw_roofline(d, k4),
                       "renv_build_ms": d["build_phases"].get("renv"),
                       "stats_dist": dist_of(dst)}
        if d.get("latency_ms"):
            lt = sorted(d["latency_ms"])
            line["dtw"]["latency"] = {"queries": len(lt), "p50_ms": lt[len(lt) // 2],
                                      "p99_ms": lt[min(len(lt) - 1, int(0.99 * len(lt)))]}
    if world == 1 and not args.no_cpu and not args.rows:
        line["build_c2"] = build_split(args, dev, stream)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, args, dev, "ED" if cfg["reach"] is None else "DTW")
    if rank == 0 and args.dump_results:
        import numpy as np
        np.savez(args.dump_results, d2=main["last"]["d2"].double().numpy(), gid=main["last"]["gid"].long().numpy())
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def reference(args):
    """The reference arm for this tier: the CPU oracle on the host cores, rank 0 only, each step
    one query over the same bounded row sample cpu_baseline uses, scaled to the collection."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import datagen
    cname = args.config or ("c3" if args.mode == "ed" else "c4")
    cfg = dict(CONFIGS[cname])
    if args.rows:
        cfg["N"] = args.rows
    if args.mode == "dtw" and cfg["reach"] is None:
        cfg["reach"] = 25
    rows = oracle_sample_size(cfg)
    try:
        import torch
        dev = torch.device("cuda") if torch.cuda.is_available() else None
    except Exception:
        dev = None
    Xh = _sample_rows(cfg, rows, dev)
    Qh = datagen.walks_cpu(0, args.warmup + args.steps, cfg["n"], seed=datagen.QUERY_SEED)
    cores = len(os.sched_getaffinity(0))
    for i in range(args.warmup):
        _oracle_time(cfg, Xh, Qh[i:i + 1], cores)
    dt = sum(_oracle_time(cfg, Xh, Qh[args.warmup + i:args.warmup + i + 1], cores) for i in range(args.steps))
    scale = cfg["N"] / rows
    value = args.steps / (dt * scale)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * scale * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded random walks, z-normalised)",
            "config": arm_config(cfg, args, world, args.queries or cfg["Q"]),
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"each step: 1 query over the first {rows:,} of {cfg['N']:,} rows "
                                       f"({dt:.2f} s measured over {args.steps} steps), time scaled x{scale:g} to "
                                       f"the full collection"},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
