"""bench.py -- SNN (arXiv 2212.07679) hot path on B200: index build + batched radius
queries, BASELINE.json metric "radius queries/s at n=1M; index build ms; % of roofline".

A step = one pass of the whole hot path over one batch: snn_build (Algorithm 1: mean,
power-iteration v1, keys, radix sort, gather + norms) + snn_query_self (Algorithm 2 for
all n points: windows, count pass, scan, write pass into CSR) + freeing both, on
BASELINE.json configs[1] (n = 1,000,000, d = 3, fp32, self-query, R from
workloads/radii.json).  Inputs are resident in HBM; L2 (126 MB) is flushed by writing a
256 MB buffer before every timed step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl snn|reference] [--config c2]

Multi-GPU (torchrun, one rank per GPU): the ranks split ONE query set (default; strong
scaling): every rank builds the replicated index and runs snn_query_*_part -- contiguous,
work-balanced ranges of key-sorted query blocks; a partitioned self-query stays symmetric
(each unordered pair once; ghost blocks before a part supply its rows' mirrored entries) --
and one all-gather of the per-part nnz rebases the parts into one global CSR
(paper_2212_07679_b200/shard.py).  ``--replicas`` (and DBSCAN, which has no cross-shard
merge) runs an independent replica per rank instead (weak scaling).  Timings are the max
over ranks.  ``--impl reference`` times the CPU oracle (fp64 brute force) on a bounded
sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "radius queries/s at n=1M (index build + self-queries)"
METRIC_DBSCAN = "DBSCAN points/s (index build + DBSCAN, n=2M)"


# ----------------------------------------------------------------------------- helpers
def load_peaks():
    try:
        return json.load(open(PEAKS_PATH)), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def fp32_alu_peak_tflops(sm_mhz: float, sms: int = 148) -> float:
    """FP32 FMA issue peak: SMs x 128 FP32 lanes x 2 flop x clock (B200_PROFILING.md
    table: 148 SMs, 1965 MHz max; 4 SMSPs x 32 lanes per SM)."""
    return sms * 128 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None
        self.path = os.path.join("/tmp", f"snn_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.QUERY}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, t0: float, t1: float):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        rows = []
        import datetime
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            rows.append((ts, parts))
        inwin = [p for ts, p in rows if t0 - 0.05 <= ts <= t1 + 0.05] or [p for _, p in rows[-3:]]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, smax = [], []
        for p in inwin:
            try:
                sm.append(float(p[2]))
                smax.append(float(p[3]))
            except ValueError:
                pass
            for k, nm in enumerate(names):
                if p[6 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(inwin)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_units(per_rank_units: int, world: int) -> int:
    """Whole-job units for weak scaling: every rank processes its own replica."""
    return per_rank_units * world


def workload(name: str):
    w = workloads.CONFIGS[name]()
    if w.R is None:
        raise SystemExit(f"radius for {name} missing: run scripts/select_radii.py")
    return w


# ----------------------------------------------------------------------------- oracle
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample_rate(w, target_s: float):
    """Oracle (fp64 brute force, host cores) on a bounded sample of the workload: returns
    (units/s, sample size, seconds, threads, sample description).

    Radius queries: the first k queries against all n points (``oracle.radius_query``).
    DBSCAN (config 5): the eps-neighbourhood counts of the first k points against all n
    points (``oracle.neighbour_counts``) -- the first of the brute-force DBSCAN's passes, so
    the rate is an upper bound on the oracle's DBSCAN points/s."""
    import oracle
    dbscan = w.dbscan_min_pts is not None

    def run(k):
        if dbscan:
            oracle.neighbour_counts(w.X, w.R, np.arange(k))
        else:
            oracle.radius_query(w.X, w.queries[:k], w.R)
    k = min(64, w.m)
    t = time.perf_counter()
    run(k)
    dt = time.perf_counter() - t
    k2 = int(min(w.m, max(k, k * target_s / max(dt, 1e-6))))
    t = time.perf_counter()
    run(k2)
    dt2 = time.perf_counter() - t
    if dbscan:
        sample = (f"eps-neighbourhood counts of the first {k2} of {w.n} points vs all {w.n} points "
                  f"(the brute-force DBSCAN's first pass; upper bound on its points/s), fp64 ({dt2:.1f} s)")
    else:
        sample = f"first {k2} of {w.m} queries vs all {w.n} points, fp64 brute force ({dt2:.1f} s)"
    return k2 / dt2, k2, dt2, oracle.num_threads(), sample


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    w = workload(args.config)
    dbscan = w.dbscan_min_pts is not None
    # per-step sample sized so the whole --steps/--warmup run ends in ~1-2 minutes
    rate, _, _, threads, _ = oracle_sample_rate(w, 2.0)
    per_step = int(max(8, min(w.m, rate * 60.0 / max(1, args.steps + args.warmup))))

    def run(s0, k):
        if dbscan:
            oracle.neighbour_counts(w.X, w.R, np.arange(s0, s0 + k))
        else:
            oracle.radius_query(w.X, w.queries[s0:s0 + k], w.R)
    for i in range(args.warmup):
        run(0, per_step)
    t = time.perf_counter()
    for i in range(args.steps):
        run((i * per_step) % max(1, w.m - per_step + 1), per_step)
    dt = time.perf_counter() - t
    value = per_step * args.steps / dt
    if dbscan:
        sample = (f"eps-neighbourhood counts of {per_step} of {w.n} points per step vs all {w.n} points "
                  f"(fp64 brute force; the DBSCAN oracle's first pass, an upper bound on its points/s)")
    else:
        sample = (f"{per_step} of {w.m} queries per step against all {w.n} points "
                  f"(fp64 brute force, no index build)")
    unit = "points/s" if dbscan else "queries/s"
    line = {"impl": "reference", "metric": METRIC_DBSCAN if dbscan else METRIC, "value": value, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(w, args),
            "cpu_baseline": {"value": value, "unit": unit, "cores": threads,
                             "kind": "oracle", "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(w, args):
    return {"workload": f"{args.config}: n={w.n}, d={w.d}, "
                        f"{'self-query' if w.Q is None else f'm={w.m} queries'}, R={w.R:.6g}",
            "n": w.n, "m": w.m, "d": w.d, "R": w.R, "input_dtype": str(w.X.dtype),
            "l2": "flushed (256 MB write) before every timed step",
            "parallelism": (f"replicas x{args.gpus} (weak scaling)" if (args.gpus <= 1 or args.replicas or w.dbscan_min_pts is not None)
                            else f"query shards x{args.gpus} (snn_query_*_part, symmetric self-query split, "
                                 f"nnz all-gather rebase; strong scaling)")}


# ----------------------------------------------------------------------------- roofline
def roofline_block(args, w, prof, times, dev, info):
    """Roofline of the dominant kernel, from CUDA-event times taken by the library on the
    launching stream (snn_profile_*) during the timed steps.

    d <= 8 : K8 scan pass (window_lowd / window_lowd_2q), FP32-ALU bound: (3d-1) flop per evaluated pair
             (eq:ip1) vs 148 SMs x 128 lanes x 2 x sm_max_mhz.
    d >= 32: K9 tcgen05 TF32 filter (tc_window_kernel), tensor bound: 2 kpad flop per pair
             (the X(J,:)^T x_q contraction) vs TF32 dense peak = measured
             bf16 burst x 1/2 (B200_PROFILING.md nominal ratio tf32 1.1 : bf16 2.25 PF).
    """
    import torch
    peaks, src = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fam = "window_count"
    if prof.get("dbscan_union", {}).get("ms", 0.0) > prof["window_count"]["ms"]:
        fam = "dbscan_union"   # DBSCAN: the union pass dominates once the counts exit early
    kms = prof[fam]["ms"]
    klaunch = prof[fam]["launches"]
    kunits = prof[fam]["units"]
    traffic = None
    try:
        tr = json.load(open(TRAFFIC_PATH))
        traffic = tr.get(args.config, {}).get("dominant_kernel_dram_bytes_per_launch")
    except Exception:
        pass
    if info.get("tc_operand", 0):
        f16 = info["tc_operand"] == 1
        kpad = info["tc_kpad"]
        flop_per_pair = 2 * w.d
        if f16:
            peak = float(peaks.get("bf16_tflops", 1590.0))
            kernel = "tc_window_kernel<F16=true> (K9 tcgen05 kind::f16 filter)"
            peak_src = f"FP16 dense = measured bf16_tflops {peaks.get('bf16_tflops')} (same tensor rate; {src})"
        else:
            peak = float(peaks.get("bf16_tflops", 1590.0)) * 0.5
            kernel = "tc_window_kernel<F16=false> (K9 tcgen05 kind::tf32 filter)"
            peak_src = f"TF32 dense = measured bf16_tflops {peaks.get('bf16_tflops')} x 0.5 (nominal 1.1 : 2.25 PF; {src})"
        bound = "tensor"
        work = (f"2d = {flop_per_pair} flop per evaluated pair (PAPER.md:216 expanded-form inner product; "
                f"the MMA runs K = {kpad}, i.e. {2 * kpad} flop incl. padding)")
    else:
        flop_per_pair = 3 * w.d - 1
        peak = fp32_alu_peak_tflops(sm_max, n_sm)
        import paper_2212_07679_b200 as snn
        snap = snn.snn_get_option("union_snap") > 0 and w.X.dtype == np.float32 and w.d <= 8
        o2q = snn.snn_get_option("scan2q")   # 0 = auto: on for d >= 2 (api.cu query_impl)
        twoq = w.X.dtype == np.float32 and w.d <= 8 and (o2q > 0 or (o2q == 0 and w.d >= 2))
        kernel, bound = ((f"union_snap_kernel<{w.d}> (K12 DBSCAN union pass, staged root snapshot)" if snap
                          else f"window_lowd<float,{w.d},union> (K12 DBSCAN union pass)") if fam == "dbscan_union"
                         else (f"window_lowd_2q<{w.d}> (K8 scan pass, two queries per thread)" if twoq
                               else f"window_lowd<float,{w.d},scan> (K8 scan pass)")), "alu"
        peak_src = f"FP32 FMA issue peak at {sm_max:.0f} MHz x {n_sm} SMs (sm_max_mhz, {src})"
        work = f"{flop_per_pair} flop per evaluated candidate pair (eq:ip1)"
    achieved = (flop_per_pair * kunits / klaunch) / (kms / klaunch * 1e-3) / 1e12 if klaunch else 0.0
    # the secondary (non-binding) roofline SURVEY.md §8(d) asks for: the same kernel's ncu DRAM
    # bytes per launch over its measured duration, against the measured copy bandwidth
    hbm = None
    if traffic and klaunch:
        gbps = traffic / (kms / klaunch * 1e-3) / 1e9
        hbm_peak = float(peaks.get("hbm_gbs", 0.0) or 0.0)
        hbm = {"achieved_gbps": gbps, "peak_gbps": hbm_peak or None,
               "frac": gbps / hbm_peak if hbm_peak else None,
               "note": "ncu dram bytes per launch (cold, serialised capture) / live kernel time; not binding"}
    return {"kernel": kernel, "bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": traffic, "hbm": hbm, "peak_source": peak_src,
            "work": f"{work}; {kunits / max(klaunch, 1):.4g} pairs per launch",
            "kernel_ms_per_launch": kms / max(klaunch, 1),
            "share_of_step": kms / sum(times) if times else None}


def step_footprint(w, nnz: int) -> int:
    """Device memory three overlapping steps may hold (staged input, index copies, result,
    workspace): what bench.py reserves in the library's pool before a timed loop."""
    x = w.X.nbytes + (0 if w.Q is None else w.Q.nbytes)
    res = (w.m + 1) * 8 + 2 * 8 * (nnz or 0)
    return int(min(3 * (4 * x + 3 * res) + (1 << 30), 48 << 30))


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    import paper_2212_07679_b200 as snn
    snn.load_library()
    for kv in args.opt:   # tuning A/B: --opt key=value (snn_set_option)
        k, v = kv.split("=")
        snn.snn_set_option(k, int(v))
    w = workload(args.config)
    X = torch.from_numpy(w.X).to(dev)
    Qd = None if w.Q is None else torch.from_numpy(w.Q).to(dev)
    R = w.R
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    dbscan = w.dbscan_min_pts is not None
    # N > 1: one query set split across the ranks (strong scaling) unless --replicas;
    # DBSCAN (config 5) has no cross-shard union-find merge: replicas
    shard = world > 1 and not dbscan and not args.replicas
    if shard:
        from paper_2212_07679_b200 import shard as shard_mod
    labels_d = torch.empty(w.n, dtype=torch.int32, device=dev) if dbscan else None

    def step():
        idx = snn.snn_build(X)
        if dbscan:   # config 5: build + DBSCAN
            k = snn.snn_dbscan(idx, R, w.dbscan_min_pts, labels_d)
            snn.snn_free(idx)
            return k
        if shard:   # this rank's work-balanced share of one query set
            r = (snn.snn_query_self_part(idx, R, rank, world) if Qd is None
                 else snn.snn_query_radius_part(idx, Qd, R, rank, world))
        else:
            r = snn.snn_query_self(idx, R) if Qd is None else snn.snn_query_radius(idx, Qd, R)
        nnz = snn.snn_result_csr(r)["nnz"]
        if shard:   # rebase: every part's first global entry (one all-gather of the part sizes)
            _, total, _ = shard_mod.part_bases(nnz, device=dev)
            nnz = total
        snn.snn_result_free(r)
        snn.snn_free(idx)
        return nnz

    # the library's stream-ordered pool keeps freed memory; reserve one step's footprint
    # before the timed loop (as before the end-to-end loops), or the first timed steps pay
    # the pool's growth (config 4: builds of 7-37 ms until ~10 GB are pooled, 2.2 ms after)
    nnz = step()
    snn.snn_pool_reserve(step_footprint(w, nnz))
    for _ in range(max(3, args.warmup)):
        nnz = step()
    _idx = snn.snn_build(X)
    info = snn.snn_index_info(_idx)
    snn.snn_free(_idx)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    snn.snn_profile_enable(True)
    l0 = snn.snn_launch_count()
    clk = ClockSampler(torch.cuda.current_device() if world == 1 else local)
    clk.start()
    time.sleep(0.3)
    t_host0 = time.time()
    times = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    t_host1 = time.time()
    clocks = clk.stop(t_host0, t_host1)
    launches = snn.snn_launch_count() - l0
    prof = {f: snn.snn_profile_read(f)
            for f in ("build", "window_count", "window_write", "query", "dbscan", "dbscan_union")}
    overflow = snn.snn_profile_read("overflow")["units"]
    lost = snn.snn_profile_read("lost")["units"]
    snn.snn_profile_enable(False)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    total_ms = max_over_ranks(sum(times), world, dev)
    units = w.m * args.steps if shard else weak_units(w.m * args.steps, world)
    value = units / (total_ms / 1e3)

    # ---- end to end through the C ABI with HOST buffers (copies inside the timed region)
    Xh = torch.from_numpy(w.X).pin_memory()
    Qh = None if w.Q is None else torch.from_numpy(w.Q).pin_memory()
    off_h = torch.empty(w.m + 1, dtype=torch.int64).pin_memory()
    idx_h = torch.empty(1 if dbscan else max(nnz, 1), dtype=torch.int32).pin_memory()
    dist_h = torch.empty(1 if dbscan else max(nnz, 1), dtype=torch.float32).pin_memory()
    labels_h = torch.empty(w.n, dtype=torch.int32).pin_memory() if dbscan else None
    snn.snn_pool_reserve(step_footprint(w, nnz))
    e2e_times = []
    for i in range(args.warmup + args.steps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        idx = snn.snn_build(Xh)
        if dbscan:
            snn.snn_dbscan(idx, R, w.dbscan_min_pts, labels_h)
        else:
            if shard:
                r = (snn.snn_query_self_part(idx, R, rank, world) if Qh is None
                     else snn.snn_query_radius_part(idx, Qh, R, rank, world))
            else:
                r = snn.snn_query_self(idx, R) if Qh is None else snn.snn_query_radius(idx, Qh, R)
            snn.snn_result_copy(r, off_h, idx_h, dist_h)
            if shard:
                shard_mod.part_bases(snn.snn_result_csr(r)["nnz"], device=dev)
            snn.snn_result_free(r)
        snn.snn_free(idx)
        e1.record()
        e1.synchronize()
        if i >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1))
    e2e_serial_ms = max_over_ranks(sum(e2e_times), world, dev)
    e2e_ms, e2e_mode = e2e_serial_ms, "serial: every step's H2D, build, query and D2H back to back"
    e2e_pipelined_ms = None
    if not dbscan:
        # pipelined: step k's CSR copy-out (snn_result_copy_async on a copy stream, into one of
        # two pinned host buffer sets) runs under step k+1's H2D + build + query; the timed
        # region ends when the last step's copy has landed in host memory
        off_h2 = torch.empty_like(off_h).pin_memory()
        idx_h2 = torch.empty_like(idx_h).pin_memory()
        dist_h2 = torch.empty_like(dist_h).pin_memory()
        bufs = [(off_h, idx_h, dist_h), (off_h2, idx_h2, dist_h2)]
        # two non-blocking streams (compute, copy): the legacy default stream would order
        # the compute behind the copies
        comp = torch.cuda.Stream(device=dev)
        cs = torch.cuda.Stream(device=dev)
        # room for three steps' results, indexes and workspaces in the library's memory pool
        snn.snn_pool_reserve(step_footprint(w, nnz), comp)
        pending = []
        ev_start = torch.cuda.Event(enable_timing=True)
        tl = [] if os.environ.get("SNN_BENCH_TIMELINE") else None   # diagnostics: per-step stream timeline
        torch.cuda.synchronize()
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                for rr, ev in pending:
                    ev.synchronize()
                    snn.snn_result_free_async(rr, comp)
                pending = []
                torch.cuda.synchronize()
                if world > 1:
                    torch.distributed.barrier()
                ev_start.record(comp)
            if tl is not None:
                e_s = torch.cuda.Event(enable_timing=True)
                e_s.record(comp)
                h_s = time.perf_counter()
            with torch.cuda.stream(comp):
                flush.fill_(1.0)
                idx = snn.snn_build(Xh, stream=comp)
                if shard:
                    r = (snn.snn_query_self_part(idx, R, rank, world, stream=comp) if Qh is None
                         else snn.snn_query_radius_part(idx, Qh, R, rank, world, stream=comp))
                else:
                    r = (snn.snn_query_self(idx, R, stream=comp) if Qh is None
                         else snn.snn_query_radius(idx, Qh, R, stream=comp))
            if len(pending) == 2:                 # buffer set i % 2 was step i-2's: retire it
                rr, ev = pending.pop(0)
                ev.synchronize()
                snn.snn_result_free_async(rr, comp)   # reused by the compute stream's next allocations
            cs.wait_stream(comp)
            if tl is not None:
                e_c = torch.cuda.Event(enable_timing=True)
                e_c.record(cs)
            snn.snn_result_copy_async(r, *bufs[i % 2], stream=cs)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(cs)
            if tl is not None:
                tl.append((e_s, e_c, ev, time.perf_counter() - h_s))
            pending.append((r, ev))
            if shard:
                shard_mod.part_bases(snn.snn_result_csr(r)["nnz"], device=dev)
            snn.snn_free_async(idx, comp)
        last = pending[-1][1]
        last.synchronize()
        piped_ms = ev_start.elapsed_time(last)
        if tl:
            for k, (a, c, d, hs) in enumerate(tl):
                print(f"step {k}: compute from {tl[0][0].elapsed_time(a):8.2f}  copy {tl[0][0].elapsed_time(c):8.2f} -> "
                      f"{tl[0][0].elapsed_time(d):8.2f}  host {hs * 1e3:.2f} ms", file=sys.stderr)
        for rr, ev in pending:
            ev.synchronize()
            snn.snn_result_free(rr)
        piped_ms = max_over_ranks(piped_ms, world, dev)
        if piped_ms < e2e_ms:   # both schedules copy every step's input and result; report the faster
            e2e_ms = piped_ms
            e2e_mode = ("pipelined: step k's D2H copy (snn_result_copy_async, copy stream, double-buffered "
                        "pinned host CSR) overlaps step k+1's H2D + build + query")
        e2e_pipelined_ms = piped_ms
    e2e_value = (w.m * args.steps if shard else weak_units(w.m * args.steps, world)) / (e2e_ms / 1e3)
    # bytes per step of the whole job: replicas copy everything on every rank; shards copy
    # X (replicated build) and the offsets on every rank, each entry once (nnz = all parts)
    h2d = (w.X.nbytes + (0 if w.Q is None else w.Q.nbytes)) * world
    d2h = (w.n * 4 if dbscan else (w.m + 1) * 8 + nnz * 8) * (1 if world == 1 else world)
    if shard:
        d2h = (w.m + 1) * 8 * world + nnz * 8
    metric = METRIC_DBSCAN if dbscan else METRIC
    unit = "points/s" if dbscan else "queries/s"

    roofline = roofline_block(args, w, prof, times, dev, info)

    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if shard else "weak", "vs_baseline": None,
            "dtype": "f64" if w.X.dtype == np.float64 else "f32", "data": "synthetic",
            "config": config_block(w, args),
            "build_ms": prof["build"]["ms"] / max(1, prof["build"]["launches"]),
            "query_ms": prof["query"]["ms"] / max(1, prof["query"]["launches"]),
            ("clusters" if dbscan else "nnz"): nnz, "overflow_records": overflow, "fix_items": lost,
            "breakdown_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()},
            "clocks": clocks, "gpu_launches": launches,
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps, "mode": e2e_mode,
                    "serial_ms_per_step": e2e_serial_ms / args.steps,
                    "pipelined_ms_per_step": None if e2e_pipelined_ms is None else e2e_pipelined_ms / args.steps},
            "roofline": roofline}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, k, dt, threads, sample = oracle_sample_rate(w, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": unit, "cores": threads,
                                "kind": "oracle", "cpu": cpu_model(), "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="snn", choices=["snn", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--cpu-seconds", type=float, default=25.0)   # the 64-query probe overestimates: ~10-15 s real
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (A/B runs)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: every rank runs its own replica (weak scaling) instead of splitting one query set")
    ap.add_argument("--shard", action="store_true", help="(default for N>1; kept for compatibility)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
