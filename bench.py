#!/usr/bin/env python3
"""bench.py — BASELINE config 2 on the B200 engine (and the reference arm).

Workload (BASELINE.json configs[1]): W1-W3 x RPS 1..20 x (static caps
10..100:10 + SABER-USL) x 64 seeds, n = 100 requests per trajectory, default
engine (usl(100, 0.05, 0.001), prefill 2000 tok/s), window 8, tick 0.01 s.
One step = one full sweep = 42,240 trajectories (per GPU; weak scaling: at N
GPUs the job is the same sweep over 64*N seeds, rows strided across ranks,
then the NCCL all-reduce that gathers every row for the summary).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

Prints ONE JSON line (rank 0).  `value` = trajectories/s with inputs resident
in HBM (CUDA events, L2 flushed between steps, max over ranks); `e2e` = the
same metric through the one-shot C-ABI call with host buffers.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# calibrate(profile(EngineConfig{}, {w3, n=1000, seed 42}, 50)).best
CAL_USL = (99.999999999997357, 0.049999999999992085, 0.0010000000000001078)
RPS = [float(r) for r in range(1, 21)]
CAPS = list(range(10, 101, 10))
MIXES = ["w1", "w2", "w3"]
N_REQ = 100
SEEDS_PER_GPU = 64
BASE_SEED = 42
WORKLOAD = ("config2: W1-W3 x RPS 1-20 x (static caps 10..100:10 + SABER-USL) x 64 seeds/GPU, "
            "n=100 requests, default engine usl(100,0.05,0.001), prefill 2000, window 8, tick 0.01")
METRIC = "simulated admission decisions/sec and sweep trajectories/sec vs CPU ref, same goodput"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ------------------------------------------------------------------ clocks --
class NvmlClockSampler:
    """SM clock and clock-event reasons sampled through NVML every ~2 ms on a
    background thread (the nvidia-smi loop below samples at ~10 Hz at best,
    i.e. once or twice in a ~140 ms timed region)."""

    def __init__(self, device):
        import pynvml as nv
        self.nv = nv
        nv.nvmlInit()
        self.h = nv.nvmlDeviceGetHandleByIndex(device)
        self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        self.samples = []
        self.skip = 0
        self.run = False
        self.thread = None

    def _loop(self):
        import time as _t
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while self.run:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                reasons = get_reasons(self.h)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((sm, reasons, util))
            except Exception:  # noqa: BLE001 (sampling is best effort)
                pass
            _t.sleep(0.002)

    def start(self):
        import threading
        self.run = True
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def mark(self):
        self.skip = len(self.samples)

    def stop(self):
        self.run = False
        if self.thread:
            self.thread.join(timeout=5)
        nv = self.nv
        names = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        got = self.samples[self.skip:] or self.samples[-1:]
        reasons = sorted({n for _, r, _ in got for n, bit in names.items() if r & bit})
        sm = [c for c, _, _ in got]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(got), "source": "NVML, ~2 ms period"}


def make_clock_sampler(device):
    try:
        return NvmlClockSampler(device)
    except Exception:  # noqa: BLE001 (no NVML: nvidia-smi loop)
        return ClockSampler(device)


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, util, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                s, m, u = float(f[1]), float(f[2]), float(f[4])
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            util.append(u)
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ host / config --
def host_info():
    """CPU model, SMT state and logical core count of the box."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    smt = None
    try:
        smt = open("/sys/devices/system/cpu/smt/active").read().strip() == "1"
    except OSError:
        pass
    return {"cpu_model": model, "smt": smt, "logical_cores": os.cpu_count()}


def bench_config(world):
    """The workload both arms report (key-identical, so the driver can match
    them): config 2 over 64 seeds per GPU."""
    return {"workload": WORKLOAD, "trajectories_per_step": len(MIXES) * len(RPS) * (len(CAPS) + 1) *
            SEEDS_PER_GPU * world, "seeds": SEEDS_PER_GPU * world, "n_gpus": world}


# -------------------------------------------------------------- reference --
def reference_sample(seeds, jobs=0):
    """Time oracle/_ref (the unmodified reference compiled from its sources)
    running saber::sweep on `seeds` seeds of the same grid, all host cores."""
    import oracle as O  # noqa: E402  (CPU-baseline / reference arm only)
    ref = O.Oracle("reference")
    base = reference_base(O, seeds)
    t0 = time.perf_counter()
    r = ref.sweep(base, MIXES, RPS, CAPS, True, seeds, jobs=jobs)
    dt = time.perf_counter() - t0
    return r, dt


def reference_base(O, seeds):
    base = O.make_config(mix="w3", n=N_REQ, seed=BASE_SEED, model=(O.USL, CAL_USL), gt=O.DEFAULT_GT)
    base.has_model = 1
    return base


def reference_arm(args):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # noqa: E402
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", args.gpus)
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    rows_per_seed = len(MIXES) * len(RPS) * (len(CAPS) + 1)
    # each step: the first 64 seeds of the workload (rank 0's shard at N = 1;
    # a bounded sample of it at N > 1), saber::sweep on every host thread
    seeds = SEEDS_PER_GPU
    for _ in range(args.warmup):
        reference_sample(seeds)
    times = []
    for _ in range(args.steps):
        _, dt = reference_sample(seeds)
        times.append(dt)
    rows = rows_per_seed * seeds
    value = rows * args.steps / sum(times)
    # decisions of the same trajectories (untimed): the reference's run() over
    # the sample's cells (saber::sweep returns no decision data)
    dec, _ = O.sweep_decisions(reference_base(O, seeds), MIXES, RPS, CAPS, True, seeds)
    decisions = float(dec.sum())
    sample = (f"{seeds} seed(s) x {rows_per_seed} cells = {rows} trajectories per step "
              f"(saber::sweep jobs=0 -> {cores} threads)")
    line = {"metric": METRIC, "value": value, "unit": "traj/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate(): mt19937_64 Poisson arrivals, task/length draws; "
                    f"seeds {BASE_SEED}..{BASE_SEED + seeds - 1})",
            "config": bench_config(world),
            "impl": "reference",
            "decisions_per_s": decisions * args.steps / sum(times),
            "decisions_per_step": decisions,
            "host": host_info(),
            "cpu_baseline": {"value": value, "unit": "traj/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "traj/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ engine --
def algorithmic_fp64_ops(rows):
    """SURVEY §8(d) W_traj summed over rows: per pass 3 + 11 per decode slot +
    4 per prefill slot; per tick 1 + 6 per high-tier entry + 6 per gate
    candidate + 1 per ledger entry scanned."""
    r = rows
    return float(np.sum(3 * r["passes"] + 11 * r["decode_updates"] + 4 * r["prefill_updates"] +
                        r["ticks"] + 6 * r["refresh_entries"] + 6 * r["gate_candidates"] +
                        r["ledger_scanned"]))


def issue_roofline(prof, sim_ms, sm_count, clk):
    """K1's limiter roofline: instruction issue.  achieved = the
    warp instructions one sweep's two trajectory kernels issue (counted by ncu
    in the committed capture of this build, profiles/sim_kernel_traffic.json;
    the work is deterministic, so the count is a property of the build and the
    workload) / their live CUDA-event time; peak = 4 schedulers x SMs x the SM
    clock sampled during the timed region (one warp instruction per scheduler
    per cycle)."""
    if not prof or "kernels" not in prof:
        return None
    inst = sum(k["warp_instructions"] for k in prof["kernels"].values())
    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz")
    if not mhz:
        return None
    achieved = inst / (sim_ms / 1e3) / 1e9
    peak = 4 * sm_count * mhz * 1e6 / 1e9
    return {"achieved": achieved, "peak": peak, "unit": "Gwarp-inst/s", "frac": achieved / peak,
            "warp_instructions_per_launch": inst,
            "capture": {"tag": prof.get("tag"), "commit": prof.get("commit"),
                        "issue_pct_under_ncu": {k: v.get("issue_active_pct")
                                                for k, v in prof["kernels"].items()},
                        "threads_per_inst": {k: v.get("threads_per_inst")
                                             for k, v in prof["kernels"].items()},
                        "file": "profiles/sim_kernel_traffic.json"}}


def roofline_entry(issue, fp64_achieved, fp64_peak, fp64_ops, traffic, sim_ms, step_ms):
    """Headline: the issue roofline of K1; the algorithmic FP64
    roofline beside it."""
    fp64 = {"achieved": fp64_achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": fp64_achieved / fp64_peak if fp64_peak else None,
            "algorithmic_fp64_ops_per_launch": fp64_ops,
            "peak_source": "measured live: DFMA microbenchmark (saber_cuda_fp64_peak); "
                           "MEASURED_PEAKS.json has no FP64 entry"}
    r = {"kernel": "sim_kernel<SABER> + sim_kernel<static> (K1, concurrent)",
         "kernel_ms": sim_ms, "share_of_step": sim_ms / step_ms, "traffic": traffic}
    if issue is not None:
        r.update({"bound": "issue", "achieved": issue["achieved"], "peak": issue["peak"],
                  "unit": issue["unit"], "frac": issue["frac"], "issue": issue, "fp64": fp64,
                  "note": "K1 is issue/latency-bound: issue roofline headline (instructions "
                          "from the committed ncu capture of this build / live kernel time), "
                          "FP64 algorithmic roofline secondary (DESIGN.md §4)"})
    else:
        r.update({"bound": "fp64", "achieved": fp64_achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                  "frac": fp64["frac"], "fp64": fp64,
                  "note": "no ncu capture found: FP64 algorithmic roofline only"})
    return r


def load_profile_traffic():
    p = os.path.join(ROOT, "profiles", "sim_kernel_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def engine_arm(args):
    import torch
    import paper_2506_19677_b200 as S

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # Test hooks for the N > 1 path on a single-GPU box (never set by the
    # driver): every rank on one device, gloo instead of NCCL.
    if os.environ.get("SABER_BENCH_DEVICE") is not None:
        local = env_int("SABER_BENCH_DEVICE", 0)
    backend = os.environ.get("SABER_BENCH_BACKEND", "nccl")
    # N > 1: the engine's own NCCL communicator does the final statistics
    # reduce (saber_cuda_sweep_plan_gather); torch.distributed is plumbing
    # only (barriers, the NCCL id broadcast, the max-over-ranks time).  The
    # gloo hook (two ranks on one GPU, tests only) gathers with torch instead,
    # since NCCL allows one rank per GPU.  SABER_BENCH_NCCL=1 forces the
    # engine-NCCL path at N = 1 (tests).
    multi = world > 1 or os.environ.get("SABER_BENCH_NCCL") == "1"
    engine_nccl = multi and backend == "nccl"
    dist = None
    if multi:
        import torch.distributed as dist  # noqa: F811
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
    device = torch.cuda.current_device()
    stream = torch.cuda.current_stream()
    comm = None
    if engine_nccl:
        uid = [S.NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = S.NcclComm(uid[0], world, rank, device)

    grid = S.SweepGrid(MIXES, RPS, CAPS, True)
    base = S.SimConfig()
    base.workload.num_requests = N_REQ
    base.model = S.SpeedModel(S.ModelFamily.Usl, CAL_USL)
    base.repeats = SEEDS_PER_GPU * world
    base.seed = BASE_SEED
    # Two plans, so consecutive sweeps pipeline: the summary of sweep k (its
    # sequential pooled sums, on a side stream) overlaps the simulation of
    # sweep k+1.  --no-pipeline runs them back to back.
    n_plans = 1 if args.no_pipeline else 2
    plans = [S.SweepPlan(grid, base, device=device, shard_index=rank, shard_count=world)
             for _ in range(n_plans)]
    views = []
    for pl in plans:
        bufs = pl.buffers()
        if multi and not engine_nccl:
            # zero-copy int64 views of the plan's row/completion buffers (gloo hook)
            views.append((torch.as_tensor(_CudaView(bufs.rows, bufs.rows_bytes), device=f"cuda:{device}"),
                          torch.as_tensor(_CudaView(bufs.completion_times, bufs.completion_bytes),
                                          device=f"cuda:{device}")))
        else:
            views.append(None)
    side = torch.cuda.Stream(device=device, priority=-1)  # high priority: summary blocks go first
    summary_done = [None] * n_plans
    root = rank == 0

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=device)

    def gather(i, strm):
        """The final statistics reduce: shards are disjoint (other ranks' rows
        are 0), so an integer sum of the raw bits onto rank 0 is an exact gather."""
        if engine_nccl:
            plans[i].gather(comm, 0, strm.cuda_stream)
        elif multi:
            for v in views[i]:
                dist.all_reduce(v)

    def step(k, sync):
        i = k % n_plans
        pl = plans[i]
        if sync:
            pl.run(stream.cuda_stream)
            gather(i, stream)
            if root:
                pl.summarize(stream.cuda_stream)
            else:
                stream.synchronize()
            return
        if summary_done[i] is not None:
            stream.wait_event(summary_done[i])  # plan i's buffers are free again
        pl.launch(stream.cuda_stream)  # per-row metrics stay on this stream: narrow
        # metrics blocks on the side stream displaced trajectory blocks (14.8 vs 13.6 ms)
        sim_done = torch.cuda.Event()
        sim_done.record(stream)
        side.wait_event(sim_done)
        with torch.cuda.stream(side):
            gather(i, side)
            if root:
                pl.summarize_launch(side.cuda_stream)
        e = torch.cuda.Event()
        e.record(side)
        summary_done[i] = e

    for k in range(args.warmup):
        flush.fill_(k)  # (also loads the fill kernel before the timed region)
        step(k, sync=True)  # synchronous: every warm-up sweep is error-checked
    torch.cuda.synchronize()

    clocks = make_clock_sampler(device)
    clocks.start()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for k in range(args.steps):
        if not os.environ.get("BENCH_NO_FLUSH"):
            flush.fill_(k)  # evict L2 (256 MB > 126 MB) between timed steps
        step(k, sync=args.no_pipeline)
    for e in summary_done:
        if e is not None:
            stream.wait_event(e)
    t_end.record(stream)
    torch.cuda.synchronize()
    for pl in plans:
        pl.wait()  # error flags of the last sweeps, stats
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    plan = plans[(args.steps - 1) % n_plans]
    launches_per_step = plan.stats()[2]
    sim_ms = [pl.stats()[1] for pl in plans]

    rows, _, summ, best = plan.fetch(completion=False, summary=root)
    total_rows = plan.n_rows
    value = total_rows * args.steps / (total_ms / 1e3)
    decisions = float(rows["decisions"].sum())
    mine = rows[rows["n"] > 0] if world > 1 else rows
    fp64_ops = algorithmic_fp64_ops(rows[np.arange(len(rows)) % world == rank])
    sim_avg_ms = float(np.mean(sim_ms))

    # e2e through the public API with host buffers, every step: the host
    # prologue + H2D of the step's inputs (plan reseed: per-seed generate()
    # draws into pinned staging, async upload), all device work, and the D2H
    # of the SweepResult payload (row statistics, summary, best caps) into
    # pinned host memory; pipelined over two plans like `value` (the D2H of
    # step k overlaps step k+1).  Wall clock, max over ranks.  The one-shot
    # saber_cuda_sweep (host in, host out, nothing overlapped) is reported
    # beside it.
    e2e_plans = [S.SweepPlan(grid, base, device=device, shard_index=rank, shard_count=world)
                 for _ in range(2)]
    pinned = []
    for _ in e2e_plans:
        st = torch.empty(total_rows * 4, dtype=torch.float64, pin_memory=True)
        bc = torch.empty(len(MIXES) * len(RPS), dtype=torch.int32, pin_memory=True)
        sm = torch.empty(len(MIXES) * 7, dtype=torch.float64, pin_memory=True)
        # (every result buffer pinned: a pageable destination would make the
        # async copy synchronous and serialise the host with the GPU)
        pinned.append((st, bc, st.numpy().view(S.ROW_STATS_DTYPE),
                       (S._native.saber_mix_summary * len(MIXES)).from_address(sm.data_ptr()),
                       bc.numpy().reshape(len(MIXES), len(RPS)), sm))
    done = [None, None]

    def e2e_step(k):
        i = k % 2
        pl = e2e_plans[i]
        if done[i] is not None:
            done[i].synchronize()  # plan i's previous results are on the host
        pl.reseed(BASE_SEED, stream.cuda_stream)
        pl.launch(stream.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(stream)
        side.wait_event(ev)
        gather_e2e(pl, side)
        if root:
            pl.summarize_launch(side.cuda_stream)
            _, _, stats_np, summ_c, best_np, _ = pinned[i]
            pl.fetch_stats_async(stats_np, summ_c, best_np, side.cuda_stream)
        e = torch.cuda.Event()
        e.record(side)
        done[i] = e

    def gather_e2e(pl, strm):
        if engine_nccl:
            pl.gather(comm, 0, strm.cuda_stream)
        elif multi:
            b = pl.buffers()
            with torch.cuda.stream(strm):
                for ptr, nb in ((b.rows, b.rows_bytes), (b.completion_times, b.completion_bytes)):
                    dist.all_reduce(torch.as_tensor(_CudaView(ptr, nb), device=f"cuda:{device}"))

    for k in range(args.warmup):
        e2e_step(k)
    torch.cuda.synchronize()
    for pl in e2e_plans:
        pl.wait()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        e2e_step(args.warmup + k)
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - t0
    for pl in e2e_plans:
        pl.wait()
    h2d, d2h = e2e_plans[0].last_h2d_bytes, e2e_plans[0].last_d2h_bytes
    if dist:
        t = torch.tensor([e2e_wall], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall = float(t.item())
    e2e_value = total_rows * args.steps / e2e_wall
    e2e_same = None
    if root:
        last = pinned[(args.warmup + args.steps - 1) % 2][2]
        e2e_same = all(np.array_equal(last[f].view(np.uint64), rows[f].astype(np.float64).view(np.uint64))
                       for f in ("goodput", "ratio_mean", "ratio_std", "cv"))
    for pl in e2e_plans:
        pl.close()
    one_shot = None
    if not multi:
        ts = []
        for k in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            _one_shot(S, grid, base, device)
            torch.cuda.synchronize()
            if k >= args.warmup:
                ts.append(time.perf_counter() - t1)
        one_shot = total_rows * len(ts) / sum(ts)

    peak = S.fp64_peak_tflops(device)
    sm_count = torch.cuda.get_device_properties(device).multi_processor_count
    achieved = fp64_ops / (sim_avg_ms / 1e3) / 1e12
    traffic, prof = load_profile_traffic()

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(rows, summ, best, base)
        line = {
            "metric": METRIC, "value": value, "unit": "traj/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate(): mt19937_64 Poisson arrivals, task/length draws; "
                    f"seeds {BASE_SEED}..{BASE_SEED + base.repeats - 1})",
            "config": bench_config(world),
            "execution": {"l2": "flushed between steps (256 MB write)",
                          "parallelism": f"rows strided over {world} GPU(s)",
                          "pipelining": "none" if args.no_pipeline else
                          "2 plans: summary of sweep k overlaps the simulation of sweep k+1"},
            "host": host_info(),
            "decisions_per_s": decisions * args.steps / (total_ms / 1e3),
            "decisions_per_step": decisions,
            "e2e": {"value": e2e_value, "unit": "traj/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "SweepPlan reseed (host prologue + async H2D) -> launch -> summarize -> "
                            "async D2H of row stats + summary into pinned memory, 2 plans in flight",
                    "results_equal_value_run": e2e_same,
                    "one_shot": {"value": one_shot, "unit": "traj/s",
                                 "path": "saber_cuda_sweep: host buffers in and out, nothing overlapped (the call reuses the previous call's device allocations; inputs are staged from the host every call)"}},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline_entry(issue_roofline(prof, sim_avg_ms, sm_count, clk), achieved, peak,
                                       fp64_ops, traffic, sim_avg_ms, total_ms / args.steps),
            "clocks": clk,
            "summary": {m: {"delta": summ[i].delta, "saber_mean_goodput": summ[i].saber_mean_goodput,
                            "best_static_mean_goodput": summ[i].best_static_mean_goodput}
                        for i, m in enumerate(MIXES)},
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
    for pl in plans:
        pl.close()
    if comm is not None:
        comm.close()
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def _one_shot(S, grid, base, device, results=False):
    """One saber_cuda_sweep call: host buffers in and out (what the drop-in
    saber::cuda::sweep issues, include/saber_cuda_adapter.hpp)."""
    import ctypes as C
    N = S._native
    p = S.SweepPlan.__new__(S.SweepPlan)
    # build the descriptor exactly as SweepPlan does, without creating a plan
    mix_ids = (C.c_int32 * len(grid.mixes))(*[int(m[1:]) for m in grid.mixes])
    rps = (C.c_double * len(grid.rps_list))(*grid.rps_list)
    caps = (C.c_int32 * len(grid.caps))(*grid.caps)
    d = N.saber_sweep_desc()
    d.mixes, d.n_mixes = mix_ids, len(grid.mixes)
    d.rps, d.n_rps = rps, len(grid.rps_list)
    d.caps, d.n_caps = caps, len(grid.caps)
    d.with_saber = 1
    d.num_requests = base.workload.num_requests
    d.length_jitter = base.workload.length_jitter
    d.window_size = base.scheduler.window_size
    d.tick = base.scheduler.tick
    d.has_model = 1
    d.model = S.api._model(base.model)
    d.ground_truth = S.api._model(base.engine.ground_truth)
    d.prefill_rate = base.engine.prefill_rate
    d.repeats = base.repeats
    d.seed = base.seed
    d.device = device
    d.shard_index, d.shard_count = 0, 1
    n_rows = int(N.lib().saber_cuda_sweep_rows(C.byref(d)))
    # the SweepResult payload of the reference's sweep(): per row the four
    # statistics (saber_row_stats) plus the per-mix summary and best caps
    stats = (N.saber_row_stats * n_rows)()
    summ = (N.saber_mix_summary * len(grid.mixes))()
    best = np.empty((len(grid.mixes), len(grid.rps_list)), dtype=np.int32)
    o = N.saber_sweep_out()
    o.row_stats = stats
    o.summary = summ
    o.best_cap_by_rps = best.ctypes.data_as(C.POINTER(C.c_int32))
    S.api._check(N.lib().saber_cuda_sweep(C.byref(d), C.byref(o)))
    del p
    if results:
        raw = np.ctypeslib.as_array(C.cast(stats, C.POINTER(C.c_double)), shape=(n_rows * 4,)).copy()
        sm = [[x.saber_mean_goodput, x.best_static_mean_goodput, x.delta, x.saber_pooled_cv,
               x.best_static_pooled_cv, x.saber_rps_mean_cv, x.best_static_rps_mean_cv] for x in summ]
        return raw, np.array(sm), best.copy()
    return int(o.h2d_bytes), int(o.d2h_bytes)


class _CudaView:
    """__cuda_array_interface__ over a raw device allocation (int64 words)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<i8",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _same(a, b):
    """Bitwise-equal float arrays (NaN == NaN)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return bool(a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64)))


def cpu_baseline(gpu_rows, summ, best, base):
    """The reference on the host cores: saber::sweep over the same 64 seeds
    (the whole N = 1 workload), timed; then every row's goodput / ratio mean /
    std / cv, the per-mix summary and the best caps compared bit for bit with
    the GPU's, and the decision counts and digests of 8 seeds' rows (the
    reference's run() over those cells, untimed)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import oracle as O  # noqa: F401
        if not O.reference_available():
            return None
    except ImportError:
        return None
    cores = os.cpu_count() or 1
    seeds = base.repeats
    r, dt = reference_sample(seeds)
    n = len(MIXES) * len(RPS) * (len(CAPS) + 1) * seeds
    checks = {k: _same(gpu_rows[k], r[k]) for k in ("goodput", "ratio_mean", "ratio_std", "cv")}
    gsum = np.array([[s.saber_mean_goodput, s.best_static_mean_goodput, s.delta, s.saber_pooled_cv,
                      s.best_static_pooled_cv, s.saber_rps_mean_cv, s.best_static_rps_mean_cv]
                     for s in summ])
    checks["summary"] = _same(gsum, r["summary"])
    checks["best_cap"] = bool(np.array_equal(np.asarray(best), r["best_cap"]))
    hs = 8
    dec, hsh = O.sweep_decisions(reference_base(O, hs), MIXES, RPS, CAPS, True, hs)
    idx = np.array([c * seeds + k for c in range(len(MIXES) * len(RPS) * (len(CAPS) + 1))
                    for k in range(hs)])
    checks["decisions"] = bool(np.array_equal(gpu_rows["decisions"][idx], dec))
    checks["decision_hash"] = bool(np.array_equal(gpu_rows["decision_hash"][idx].astype(np.uint64), hsh))
    return {"value": n / dt, "unit": "traj/s", "cores": cores, "kind": "reference",
            "sample": f"saber::sweep over seeds {BASE_SEED}..{BASE_SEED + seeds - 1} of the same grid "
                      f"({n} trajectories, {dt:.2f} s, jobs=0)",
            "same_goodput_rows": n, "same_goodput": checks["goodput"],
            "parity": checks, "parity_ok": all(checks.values()),
            "parity_scope": f"rows/summary/best caps: all {n}; decision counts+digests: "
                            f"{len(idx)} rows (seeds {BASE_SEED}..{BASE_SEED + hs - 1})"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="run each sweep's summary after it instead of overlapping the next sweep")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    return engine_arm(args)


if __name__ == "__main__":
    sys.exit(main())
