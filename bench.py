#!/usr/bin/env python
"""Benchmark of the B200 NFFT hot path (BASELINE.json metric / configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--m 4] [--config cfg2_1d_2e18]
    python bench.py --impl reference ...      # the CPU oracle arm

A step is one pass of the transform hot path over one batch of
synthetic input on a precomputed plan: the direct NFFT (deconvolve/pad, cuFFT,
interpolation: a4-a6) and the adjoint NFFT (spreading, cuFFT, crop/
deconvolve: a7-a9), as the paper measures transforms (precomputation is plan
setup, timed separately per SURVEY §8(d)). The node binning
+ stable sort (a1-a2) is reported as its own stage and in `with_precompute`
(the same step with nfft_precompute re-run inside it); the node-independent
window tables (a0, a3) are built at plan creation. Inputs are resident in HBM
and L2 is flushed (256 MiB write + 256 MiB read) before every timed step; each
step is timed with CUDA events on the plan stream, and the K steps sit between
a barrier + synchronize on both sides. value = units processed by all ranks /
max-over-ranks time (units: nodes, node-vectors for batches).

Multi-GPU (--gpus N; without torchrun the script launches N ranks itself):
  --mode weak      (default) one independent transform per rank, no data-path
                   collective (scaling "weak");
  --mode nodeshard one transform split by nodes, NCCL all_reduce of the outputs
                   (scaling "strong");
  --mode batch     the batch split over ranks (32/G vectors each), optionally
                   node-sharded inside groups of --node-groups ranks (config 5,
                   scaling "strong").
At N = 1, rank 0 also measures every other BASELINE config (`configs` key:
value, roofline, e2e, cpu_baseline per config; the radial configs batch-
sharded) and the m = 3..8 sweep of the 1D/2D sets (`m_sweep`).
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NFFT forward/adjoint nodes/sec (fp64, σ=2, m=4..8) and roofline fraction"
UNIT = "nodes/s"
FALLBACK_HBM = 6650.0
OTHER_CONFIGS = ("cfg3_2d_512", "cfg4_3d_64", "cfg5_radial_s2", "cfg5_radial_s125")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2_1d_2e18")
    ap.add_argument("--m", type=int, default=None, help="window half-width (default: the config's, 4)")
    ap.add_argument("--mode", default="weak", choices=["weak", "nodeshard", "batch"])
    ap.add_argument("--node-groups", type=int, default=1, help="--mode batch: ranks per node-shard group (G_n)")
    ap.add_argument("--method", default="auto")
    ap.add_argument("--precompute", default="auto", help="window strategy: auto | polynomial | tensor | full")
    ap.add_argument("--tile", default="")
    ap.add_argument("--no-sweep", action="store_true", help="skip the m = 3..8 sweep")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--no-strategies", action="store_true", help="skip the precompute-strategy table")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline measurement")
    ap.add_argument("--no-graph", action="store_true", help="launch the step kernel by kernel (no CUDA graph)")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work per cpu_baseline")
    return ap.parse_args(argv)


def peaks():
    """HBM copy bandwidth (MEASURED_PEAKS.json, driver-written) and the FMA
    peaks measured by tools/micro/fma_peak.cu (profiles/r02/fma_peak.jsonl)."""
    hbm, mhz, src = FALLBACK_HBM, 1965.0, "fallback 6650 GB/s (B200_PROFILING.md)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        hbm, mhz, src = float(d.get("hbm_gbs", FALLBACK_HBM)), float(d.get("sm_max_mhz", 1965.0)), \
            "measured hbm_gbs (MEASURED_PEAKS.json)"
    fp = {"fp64": 148 * 64 * 2 * mhz * 1e6 / 1e12, "fp32": 148 * 128 * 2 * mhz * 1e6 / 1e12,
          "source": f"derived: 148 SM x 64 FP64 / 128 FP32 FMA lanes x 2 x {mhz:.0f} MHz"}
    q = os.path.join(ROOT, "profiles", "r02", "fma_peak.jsonl")
    if os.path.exists(q):
        runs = [json.loads(l) for l in open(q) if l.strip().startswith("{")]
        if runs:
            fp = {"fp64": max(r["dfma_tflops"] for r in runs),
                  "fp32": max(max(r["ffma_tflops"], r["ffma2_tflops"]) for r in runs),
                  "source": "measured: tools/micro/fma_peak.cu (DFMA / FFMA / FFMA2 chains, all SMs), "
                            "profiles/r02/fma_peak.jsonl, at 1965 MHz"}
    return hbm, src, fp


def algorithmic(w):
    """Per-launch algorithmic bytes and flops:
    resampling: B*c*prod(Ntilde) + B*c*M + r*D*M bytes,
                2*M*[B*2*sum_{d=1..D}(2m)^d + 2m*D*deg] flops (deg = 2m, the paper's);
    deconv/pad: 2*B*c*prod N (the zero padding is written once per plan); crop: 2*B*c*prod N
    (the owner-computes spread rewrites every cell, so no re-zeroing)."""
    c = 16 if w["precision"] == "c128" else 8
    r = 8 if w["precision"] == "c128" else 4
    D, M, B, m = len(w["N"]), w["M"], w["batch"], w["m"]
    nt = int(np.prod([2 * math.ceil(w["sigma"] * n / 2) for n in w["N"]]))
    nn = int(np.prod(w["N"]))
    res_bytes = B * c * nt + B * c * M + r * D * M
    res_flops = 2 * M * (B * 2 * sum((2 * m) ** d for d in range(1, D + 1)) + 2 * m * D * (2 * m))
    return dict(resample_bytes=res_bytes, resample_flops=res_flops, deconv_bytes=2 * B * c * nn,
                crop_bytes=2 * B * c * nn, grid_cells=nt)


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    def __init__(self, device_index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle (reference arm, cpu_baseline)
# The oracle (oracle/nfft.py, plain fp64 numpy) is timed AS IT STANDS. The
# all-cores number runs it in a pool of spawned processes, one task per
# (batch vector, node chunk): each task is one oracle forward (rows = the
# chunk) + one oracle adjoint of the chunk's nodes, so every task repeats the
# full deconvolution + FFT of the grid steps.

_OW = {}


def _oracle_init(config, seed, m):
    sys.path.insert(0, ROOT)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from paper_2208_00049_b200 import workloads
    _OW["w"] = workloads.make(config, seed=seed, m=m)


def _oracle_task(args):
    b, lo, hi = args
    from oracle import nfft as onfft
    w = _OW["w"]
    nodes = w["nodes"][lo:hi].astype(np.float64)
    onfft.forward(nodes, w["fhat"][b].astype(np.complex128), w["N"], w["m"], w["sigma"])
    onfft.adjoint(nodes, w["f"][b][lo:hi].astype(np.complex128), w["N"], w["m"], w["sigma"])
    return hi - lo


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OraclePool:
    """The oracle on the host cores: a spawn pool (no CUDA state in the children)."""

    def __init__(self, config, seed, m, procs):
        import multiprocessing as mp
        self.procs = procs
        self.pool = mp.get_context("spawn").Pool(procs, initializer=_oracle_init, initargs=(config, seed, m))
        from paper_2208_00049_b200 import workloads
        self.w = workloads.make(config, seed=seed, m=m)
        self.chunk = None
        self.rep = 1

    def tasks(self, sample, batches):
        ch = self.chunk or max(1, -(-sample // self.procs))
        one = [(b, lo, min(lo + ch, sample)) for b in range(batches) for lo in range(0, sample, ch)]
        return one * self.rep

    def run(self, sample, batches):
        """One pass: forward + adjoint of the first `sample` nodes for `batches`
        vectors, in tasks of self.chunk nodes (the whole pass self.rep times,
        concurrently, when one pass has fewer tasks than processes: independent
        transforms of the same workload); returns (units, seconds)."""
        tasks = self.tasks(sample, batches)
        t0 = time.perf_counter()
        n = sum(self.pool.map(_oracle_task, tasks, chunksize=1))
        return n, time.perf_counter() - t0

    def _one(self, n):
        t0 = time.perf_counter()
        self.pool.apply(_oracle_task, ((0, 0, n),))
        return time.perf_counter() - t0

    def calibrate(self, budget_s):
        """Task size and sample (nodes x vectors) so that one pass takes about
        budget_s on the pool: per task t = t0 + n t1 (t0: the grid steps every
        oracle call repeats); tasks are made >= 4 t0 / t1 nodes where the
        workload allows, so the repeated grid steps cost <= ~20 %."""
        w = self.w
        M, B = w["M"], w["batch"]
        self.pool.map(_oracle_task, [(0, 0, 1)] * self.procs, chunksize=1)  # warm every worker
        n_small, n_big = min(M, 16), min(M, 4096)
        ts, tb = self._one(n_small), self._one(n_big)
        t1 = max((tb - ts) / max(n_big - n_small, 1), 1e-9)
        t0 = max(ts - n_small * t1, 0.0)
        self.chunk = int(min(M, max(-(-M // self.procs) if B == 1 else M, 4 * t0 / t1, 1)))
        best = (self.chunk, 1)
        for batches in range(1, B + 1):
            for sample in sorted({min(M, self.chunk * k) for k in range(1, -(-M // self.chunk) + 1)}):
                ntasks = batches * -(-sample // self.chunk)
                est = -(-ntasks // self.procs) * (t0 + min(self.chunk, sample) * t1)
                if est <= budget_s and sample * batches > best[0] * best[1]:
                    best = (sample, batches)
        # fewer tasks than processes (a small 1D step whose grid steps dominate): independent copies
        ntasks = best[1] * -(-best[0] // self.chunk)
        self.rep = max(1, self.procs // max(ntasks, 1))
        return best

    def close(self):
        self.pool.close()
        self.pool.join()


def measure_oracle(config, seed, m, budget_s, procs=None):
    procs = procs or cpu_cores()
    pool = OraclePool(config, seed, m, procs)
    try:
        sample, batches = pool.calibrate(budget_s / 2)
        units, secs, passes = 0, 0.0, 0
        while secs < budget_s / 2 or passes == 0:
            n, dt = pool.run(sample, batches)
            units += n
            secs += dt
            passes += 1
    finally:
        pool.close()
    used = min(procs, len(pool.tasks(sample, batches)))
    return {"value": units / secs, "unit": UNIT, "cores": used, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"{passes} pass(es) of the oracle (plain fp64 numpy, oracle/nfft.py) over the first {sample} of "
                      f"{pool.w['M']} nodes x {batches} of {pool.w['batch']} batch vector(s) of {config} (direct + "
                      f"adjoint NFFT; tasks of {pool.chunk} nodes, each oracle call repeating the grid deconvolution "
                      f"+ FFT; {pool.rep} concurrent cop(ies) of each pass) in {procs} spawned process(es), "
                      f"{used} busy; {secs:.1f} s",
            "seconds": secs}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2208_00049_b200 import workloads
    w = workloads.make(a.config, seed=0, m=a.m)
    w["name"] = a.config
    procs = cpu_cores()
    pool = OraclePool(a.config, 0, w["m"], procs)
    try:
        step_budget = max(0.5, min(10.0, 150.0 / max(a.steps + a.warmup, 1)))
        sample, batches = pool.calibrate(step_budget)
        for _ in range(a.warmup):
            pool.run(sample, batches)
        units, secs = 0, 0.0
        for _ in range(a.steps):
            n, dt = pool.run(sample, batches)
            units += n
            secs += dt
    finally:
        pool.close()
    value = units / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * secs / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(a, w, "reference"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(procs, len(pool.tasks(sample, batches))),
                         "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"each step = the oracle (plain fp64 numpy) on the first {sample} nodes x "
                                   f"{batches} vector(s) of the workload ({pool.rep} concurrent cop(ies)), in "
                                   f"{procs} processes"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(a, w, mode):
    par = {"weak": f"independent transform per GPU x{a.gpus}", "nodeshard": f"node shards x{a.gpus} + NCCL all_reduce",
           "batch": f"batch shards x{a.gpus // a.node_groups} x node shards x{a.node_groups}",
           "reference": "CPU oracle"}[mode]
    return {"workload": f"{w['name']}: {len(w['N'])}D N={'x'.join(map(str, w['N']))} M={w['M']} "
                        f"{'ComplexF64' if w['precision'] == 'c128' else 'ComplexF32'} sigma={w['sigma']} m={w['m']} "
                        f"batch={w['batch']}; step = the direct + adjoint NFFT on the precomputed plan (independent "
                        f"inputs; one nfft_execute, adjoint overlapping forward; the node binning/sort is plan setup, "
                        f"timed separately as in SURVEY 8(d): see with_precompute / stages_ms_mean.precompute)",
            "nodes": "uniform i.i.d. in [-1/2,1/2)^D" if "radial" not in w["name"] else
                     "golden-angle radial spokes (402 x 512)", "seed": "rank" if mode == "weak" else 0,
            "l2": "flushed before every step (256 MiB write + 256 MiB read)", "parallelism": par,
            "precompute_strategy": getattr(a, "precompute", "auto")}


# ----------------------------------------------------------------------------- our arm

class Ctx:
    pass


def setup_dist(a):
    import torch
    import torch.distributed as dist
    ctx = Ctx()
    ctx.world = int(os.environ.get("WORLD_SIZE", "1"))
    ctx.rank = int(os.environ.get("RANK", "0"))
    ctx.local = int(os.environ.get("LOCAL_RANK", "0"))
    if ctx.world != a.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={ctx.world} but --gpus {a.gpus}")
    torch.cuda.set_device(ctx.local)
    if ctx.world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", ctx.local))
    ctx.dev = torch.device("cuda", ctx.local)
    ctx.stream = torch.cuda.Stream(ctx.dev)
    ctx.flush_w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=ctx.dev)
    ctx.flush_r = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=ctx.dev)
    ctx.flush_sink = torch.empty((), dtype=torch.float32, device=ctx.dev)
    return ctx


def barrier(ctx):
    if ctx.world > 1:
        import torch.distributed as dist
        dist.barrier()


def flush(ctx):
    """L2 flush between steps: write 256 MiB (> 126 MB L2), then read another
    256 MiB so the write-back of the dirty lines also happens here."""
    ctx.flush_w.zero_()
    ctx.flush_sink.copy_(ctx.flush_r.sum())


def make_workload(a, ctx, config, mode, m):
    from paper_2208_00049_b200 import workloads
    w = workloads.make(config, seed=ctx.rank if mode == "weak" else 0, m=m)
    w["name"] = config
    return w


def build(a, ctx, w, mode, timing=False):
    """Plan (and the distributed wrapper) on this rank, precomputed; returns
    (obj, plan, fhat, f, fout, yout, units_per_rank_step, units_total_step)."""
    import torch
    import paper_2208_00049_b200 as pkg
    from paper_2208_00049_b200.dist import HybridNfft, ShardedNfft
    tile = tuple(int(x) for x in a.tile.split(",")) if a.tile else None
    kw = dict(m=w["m"], sigma=w["sigma"], precision=w["precision"], tile=tile, stream=ctx.stream.cuda_stream,
              device=ctx.local, method=a.method, timing=timing, check_nodes=False, precompute=a.precompute)
    B = w["batch"]
    with torch.cuda.stream(ctx.stream):
        nodes = torch.from_numpy(w["nodes"]).to(ctx.dev)
        if mode == "batch":
            obj = HybridNfft(nodes, w["N"], B, g_n=a.node_groups, **kw)
            b0, b1 = obj.batch_range
        elif mode == "nodeshard":
            obj = ShardedNfft(nodes, w["N"], batch=B, **kw)
            b0, b1 = 0, B
        else:
            obj = pkg.NfftPlan(nodes, w["N"], batch=B, **kw)
            b0, b1 = 0, B
        obj.precompute()
        plan = obj.plan if hasattr(obj, "plan") else obj
        fhat = torch.from_numpy(np.ascontiguousarray(w["fhat"][b0:b1])).to(ctx.dev)
        f = torch.from_numpy(np.ascontiguousarray(w["f"][b0:b1])).to(ctx.dev)
        fout = torch.zeros((b1 - b0, w["M"]), dtype=plan.tdtype_c, device=ctx.dev)
        yout = torch.empty((b1 - b0,) + tuple(w["N"]), dtype=plan.tdtype_c, device=ctx.dev)
    ctx.stream.synchronize()
    units_total = w["M"] * B * (ctx.world if mode == "weak" else 1)
    return obj, plan, fhat, f, fout, yout, units_total


def run_steps(a, ctx, w, mode, steps, warmup, staged=False, with_pre=False, seq_omit=None):
    """K timed steps (events on the plan stream, L2 flushed before each).
    Default: the step is one nfft_execute of the direct and the adjoint NFFT
    (adjoint || forward on plan-internal streams), captured as one CUDA graph;
    node/batch shards: forward + adjoint through the dist wrappers (zeroing,
    kernels, NCCL all_reduce) in the graph. with_pre: the precompute re-runs
    inside the step. staged: the seven stages one after another inside ONE
    graph with external event-record nodes between them (per-stage durations).
    seq_omit: the seven stages one after another in one graph without event
    nodes, stage seq_omit left out (-1: none) — the difference to the full
    sequence is the stage's marginal time (no event-node overhead)."""
    import torch
    obj, plan, fhat, f, fout, yout, units_total = build(a, ctx, w, mode)
    names = ["precompute", "deconv", "fft_fwd", "interp", "spread", "fft_adj", "crop"]
    stage_fns = [lambda: plan.run_stage("precompute"), lambda: plan.run_stage("fwd_deconv", fhat),
                 lambda: plan.run_stage("fwd_fft"), lambda: plan.run_stage("fwd_interp", None, fout),
                 lambda: plan.run_stage("adj_spread", f), lambda: plan.run_stage("adj_fft"),
                 lambda: plan.run_stage("adj_crop", None, yout)]
    sev = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(names) + 1)]
           for _ in range(2)] if staged else None

    def one(slot=0):
        if seq_omit is not None:
            for k, fn in enumerate(stage_fns):
                if k != seq_omit:
                    fn()
            return
        if staged:
            for k, fn in enumerate(stage_fns):
                sev[slot][k].record(ctx.stream)
                fn()
            sev[slot][len(names)].record(ctx.stream)
            return
        if mode == "weak":
            plan.execute(with_pre, fhat, fout, f, yout)
        else:
            if with_pre:
                plan.run_stage("precompute")
            obj.forward(fhat, out=fout)
            obj.adjoint(f, out=yout)

    with torch.cuda.stream(ctx.stream):
        for _ in range(warmup):
            flush(ctx)
            one(0)
    ctx.stream.synchronize()
    launches_per_step = 0
    g = None
    if not a.no_graph:
        g = torch.cuda.CUDAGraph()
        l0 = plan.launches()
        with torch.cuda.graph(g, stream=ctx.stream):
            one(1)
        launches_per_step = plan.launches() - l0
    ctx.stream.synchronize()
    l0 = plan.launches()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    stage = {n: [] for n in names} if staged else {}
    barrier(ctx)
    torch.cuda.synchronize(ctx.dev)
    with ClockSampler(ctx.local) as clk:
        for s in range(steps):
            with torch.cuda.stream(ctx.stream):
                flush(ctx)
                ev[s][0].record(ctx.stream)
                if g is not None:
                    g.replay()
                else:
                    one(1)
                ev[s][1].record(ctx.stream)
            if staged:  # the graph's event nodes are reused: read them every step
                ctx.stream.synchronize()
                for k, n in enumerate(names):
                    stage[n].append(sev[1][k].elapsed_time(sev[1][k + 1]))
        torch.cuda.synchronize(ctx.dev)
    barrier(ctx)
    launches = launches_per_step * steps if g is not None else plan.launches() - l0
    per_step = [ev[s][0].elapsed_time(ev[s][1]) for s in range(steps)]
    ms = sum(per_step)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=ctx.dev)
    if ctx.world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    del g
    features = sorted(plan.features())
    obj.close()
    return dict(ms=float(ms_t.item()), stage=stage, launches=launches, clocks=clk.summary(),
                units_total=units_total, features=features, median_ms=statistics.median(per_step),
                midmean_ms=midmean(per_step))


def roofline(w, means, step_ms, hbm, hbm_src, fp):
    """Roofline of the dominant library kernel (by mean duration inside the staged graph)."""
    alg = algorithmic(w)
    mine = {k: v for k, v in means.items() if k in ("deconv", "interp", "spread", "crop")}
    dom = max(mine, key=mine.get)
    bytes_of = {"interp": alg["resample_bytes"], "spread": alg["resample_bytes"], "deconv": alg["deconv_bytes"],
                "crop": alg["crop_bytes"]}
    flops_of = {"interp": alg["resample_flops"], "spread": alg["resample_flops"]}
    fp64 = w["precision"] == "c128"
    fpk = fp["fp64" if fp64 else "fp32"]
    t_hbm = bytes_of[dom] / (hbm * 1e9)
    t_fp = flops_of.get(dom, 0) / (fpk * 1e12)
    dom_s = means[dom] * 1e-3
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{w['name']}:m{w['m']}:{dom}")
    if t_fp > t_hbm:
        roof = {"bound": "alu", "achieved": flops_of[dom] / dom_s / 1e12, "peak": fpk, "unit": "TFLOP/s",
                "peak_source": f"{'FP64 DFMA' if fp64 else 'FP32 FFMA'} peak, {fp['source']}"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_of[dom] / dom_s / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": hbm_src}
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": traffic, "kernel": dom,
                 "algorithmic_bytes": bytes_of[dom], "algorithmic_flops": flops_of.get(dom, 0),
                 "kernel_ms_mean": means[dom], "kernel_share": means[dom] / step_ms,
                 "note": "kernel duration = marginal time of its stage in one graph of the seven stages run one "
                         "after another (interquartile-mean sequence time minus that of the sequence without the stage, "
                         "L2 flushed before each step; D >= 2 spread stage includes the value permutation "
                         "kernel)"})
    return roof


def midmean(xs):
    """Interquartile mean. CUDA event differences on this box come in ~2 us
    quanta, so a median of per-step times is quantised too; the mean over the
    middle half averages the quanta (the event phases are random from step to
    step) and still drops the flush-induced outliers."""
    xs = sorted(xs)
    k = len(xs) // 4
    mid = xs[k:len(xs) - k] or xs
    return sum(mid) / len(mid)


def measure_config(a, ctx, config, mode, steps, warmup, m=None, e2e=True, cpu=True, extra=True, with_pre=True,
                   cpu_budget=None):
    """value, roofline, stages, e2e and cpu_baseline of one config (this rank's
    view; value/ms are max over ranks)."""
    hbm, hbm_src, fp = peaks()
    w = make_workload(a, ctx, config, mode, m)
    main = run_steps(a, ctx, w, mode, steps, warmup)
    units = main["units_total"]
    value = units * steps / (main["ms"] * 1e-3)
    out = {"value": value, "unit": UNIT, "ms_per_step": main["ms"] / steps, "steps": steps, "m": w["m"],
           "gpu_launches": main["launches"], "clocks": main["clocks"], "features": main["features"],
           "dtype": "f64" if w["precision"] == "c128" else "f32", "w": w}
    if extra:
        n2 = max(10, min(steps, 50))
        st = run_steps(a, ctx, w, mode, n2, warmup, staged=True)
        means = {k: (statistics.mean(v) if v else 0.0) for k, v in st["stage"].items()}
        out["stages_ms_mean"] = means
        out["ms_per_step_sequential"] = st["ms"] / n2
        # marginal stage times: the seven-stage sequence with and without each stage (no event nodes);
        # interquartile means of the per-step times (the flush before every step makes single steps
        # noisy, and the event clock's ~2 us quantum would quantise a median)
        n3 = max(n2, 100)
        full = run_steps(a, ctx, w, mode, n3, warmup, seq_omit=-1)["midmean_ms"]
        marg = {}
        for k, name in enumerate(["precompute", "deconv", "fft_fwd", "interp", "spread", "fft_adj", "crop"]):
            marg[name] = full - run_steps(a, ctx, w, mode, n3, warmup, seq_omit=k)["midmean_ms"]
        out["stages_ms_marginal"] = marg
        out["ms_per_step_sequential_no_events"] = full
        if with_pre:
            pre = run_steps(a, ctx, w, mode, n2, warmup, with_pre=True)
            out["with_precompute"] = {"ms_per_step": pre["ms"] / n2, "value": units / (pre["ms"] / n2 * 1e-3),
                                      "unit": UNIT,
                                      "note": "step + node binning/sort (nfft_precompute) re-run every step"}
        out["precompute_nodes_per_s"] = w["M"] / (means["precompute"] * 1e-3) if means["precompute"] > 0 else None
        out["roofline"] = roofline(w, marg, main["ms"] / steps, hbm, hbm_src, fp)
    if e2e and mode == "weak":
        out["e2e"] = measure_e2e(a, ctx, w)
    if cpu and ctx.rank == 0 and ctx.world == 1:
        budget = cpu_budget or a.cpu_budget
        out["cpu_baseline"] = measure_oracle(config, 0, w["m"], budget)
        out["cpu_baseline"]["cpu_1core"] = measure_oracle(config, 0, w["m"], max(1.0, budget / 4), procs=1)
    return out


def measure_e2e(a, ctx, w, steps=None, pipe=4):
    """Same metric through the C ABI with pinned HOST buffers: per step one
    nfft_execute of the direct NFFT (host fhat -> host f) and the adjoint
    (host f -> host y) on a precomputed plan; host<->device copies are inside
    the timed region (the final event follows the downloads). As a user
    streaming independent transforms would, the steps alternate between `pipe`
    plans on their own streams (own host output buffers), so the uploads of
    step k + 1 overlap the downloads of step k on the full-duplex link."""
    import torch
    import paper_2208_00049_b200 as pkg
    steps = steps or max(6, min(a.steps, 50))

    def pinned(arr):
        t = torch.from_numpy(np.ascontiguousarray(arr)).pin_memory()
        return t, t.numpy()

    _, nodes_h = pinned(w["nodes"])
    _, fhat_h = pinned(w["fhat"])
    _, f_h = pinned(w["f"])
    tile = tuple(int(x) for x in a.tile.split(",")) if a.tile else None
    streams = [torch.cuda.Stream(ctx.dev) for _ in range(pipe)]
    plans, outs = [], []
    for k in range(pipe):
        plans.append(pkg.NfftPlan(nodes_h, w["N"], m=w["m"], sigma=w["sigma"], precision=w["precision"],
                                  batch=w["batch"], tile=tile, stream=streams[k].cuda_stream, device=ctx.local,
                                  method=a.method, check_nodes=False, precompute=a.precompute).precompute())
        outs.append((pinned(np.empty((w["batch"], w["M"]), w["f"].dtype))[1],
                     pinned(np.empty((w["batch"],) + tuple(w["N"]), w["fhat"].dtype))[1]))

    def step(i):
        k = i % pipe
        plans[k].execute(False, fhat_h, outs[k][0], f_h, outs[k][1])

    for i in range(2 * pipe):
        step(i)
    torch.cuda.synchronize(ctx.dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(ctx.stream)
    for st in streams:
        st.wait_event(t0)
    for i in range(steps):
        step(i)
    for st in streams:
        ctx.stream.wait_stream(st)
    t1.record(ctx.stream)
    t1.synchronize()
    ms = t0.elapsed_time(t1)
    for p in plans:
        p.close()
    h2d = w["fhat"].nbytes + w["f"].nbytes
    d2h = outs[0][0].nbytes + outs[0][1].nbytes
    return {"value": w["M"] * w["batch"] * steps / (ms * 1e-3) * ctx.world, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "pipeline": f"{pipe} plans on their own streams, steps alternating"}


def measure_strategies(a, ctx, steps=20, warmup=3):
    """The window precomputation strategies (the paper's Fig. 4
    compares their transform time and precomputation time):
    per config and strategy, the step throughput (direct + adjoint, as the main
    line) and the precompute time (nfft_precompute alone, L2 flushed, graph)."""
    import torch
    import argparse as _ap
    out = {}
    for config in ("cfg2_1d_2e18",) + OTHER_CONFIGS:
        w = make_workload(a, ctx, config, "weak", None)
        D, M, m = len(w["N"]), w["M"], w["m"]
        r = 8 if w["precision"] == "c128" else 4
        table = {"polynomial": 0, "tensor": M * D * 2 * m * r, "full": M * (2 * m) ** D * (r + 4)}
        out[config] = {}
        for strat in ("polynomial", "tensor", "full"):
            aa = _ap.Namespace(**vars(a))
            aa.precompute = strat
            res = run_steps(aa, ctx, w, "weak", steps, warmup)
            obj, plan, *_ = build(aa, ctx, w, "weak")
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=ctx.stream):
                plan.run_stage("precompute")
            times = []
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(ctx.stream):
                    flush(ctx)
                    e0.record(ctx.stream)
                    g.replay()
                    e1.record(ctx.stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            feats = sorted(plan.features())
            del g
            obj.close()
            out[config][strat] = {"value": res["units_total"] * steps / (res["ms"] * 1e-3), "unit": UNIT,
                                  "ms_per_step": res["ms"] / steps, "precompute_ms": statistics.median(times),
                                  "table_bytes": table[strat], "features": feats}
    return out


def relaunch(a):
    """`bench.py --gpus N` without torchrun: launch N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1 and return their exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a)
    if a.impl == "reference":
        return run_reference(a)
    if a.mode == "batch" and a.gpus % a.node_groups:
        raise SystemExit("--node-groups must divide --gpus")
    ctx = setup_dist(a)
    config = a.config
    mode = a.mode
    res = measure_config(a, ctx, config, mode, a.steps, a.warmup, m=a.m, e2e=not a.no_e2e, cpu=not a.no_cpu)
    w = res.pop("w")

    configs = None
    if not a.no_configs:
        configs = {}
        for c in OTHER_CONFIGS:
            if c == config:
                continue
            # one GPU: the plain plan (direct || adjoint in one execute); N GPUs: the radial batches split by
            # batch (x node groups), the others by nodes (strong scaling of one transform)
            cmode = "weak" if ctx.world == 1 else ("batch" if "radial" in c else "nodeshard")
            r = measure_config(a, ctx, c, cmode, max(10, min(a.steps, 40)), 3, e2e=not a.no_e2e and cmode == "weak",
                               cpu=not a.no_cpu, cpu_budget=a.cpu_budget / 2)
            r.pop("w")
            r["mode"] = cmode
            r["scaling"] = "weak" if cmode == "weak" else "strong"
            configs[c] = r

    sweep = None
    if not a.no_sweep and ctx.world == 1:
        sweep = {}
        for c in ("cfg2_1d_2e18", "cfg3_2d_512"):
            sweep[c] = {}
            for mm in range(3, 9):
                r = measure_config(a, ctx, c, "weak", 20, 3, m=mm, e2e=False, cpu=False, with_pre=False)
                sweep[c][f"m{mm}"] = {"value": r["value"], "ms_per_step": r["ms_per_step"],
                                      "interp_ms": r["stages_ms_marginal"]["interp"],
                                      "spread_ms": r["stages_ms_marginal"]["spread"], "roofline_frac": r["roofline"]["frac"],
                                      "roofline_bound": r["roofline"]["bound"]}

    strategies = None
    if not a.no_strategies and ctx.world == 1:
        strategies = measure_strategies(a, ctx)

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ctx.world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak" if mode == "weak" else "strong", "vs_baseline": None,
            "dtype": res["dtype"], "data": "synthetic", "config": config_dict(a, w, mode),
            "roofline": res["roofline"], "cpu_baseline": res.get("cpu_baseline"), "e2e": res.get("e2e"),
            "gpu_launches": res["gpu_launches"], "clocks": res["clocks"], "features": res["features"],
            "stages_ms_mean": res["stages_ms_mean"], "ms_per_step_sequential": res["ms_per_step_sequential"],
            "stages_ms_marginal": res["stages_ms_marginal"],
            "ms_per_step_sequential_no_events": res["ms_per_step_sequential_no_events"],
            "with_precompute": res.get("with_precompute"), "precompute_nodes_per_s": res["precompute_nodes_per_s"],
        }
        if configs:
            line["configs"] = configs
        if sweep:
            line["m_sweep"] = sweep
        if strategies:
            line["strategies"] = strategies
        print(json.dumps(line), flush=True)
    if ctx.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
