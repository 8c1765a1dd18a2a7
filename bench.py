#!/usr/bin/env python
"""Benchmark of the B200 NFFT hot path (BASELINE.json metric / configs[1]).

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
and L2 is flushed (256 MiB write) before every timed step; each step is timed
with CUDA events on the plan stream, and the K steps sit between a barrier +
synchronize on both sides. value = nodes processed by all ranks / max-over-
ranks time. N > 1 (torchrun): weak scaling, one independent transform per
rank, no data-path collective (--mode nodeshard: one transform split by nodes
with an NCCL all_reduce, strong scaling).
"""

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NFFT forward/adjoint nodes/sec (fp64, σ=2, m=4..8) and roofline fraction"
UNIT = "nodes/s"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2_1d_2e18")
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--mode", default="weak", choices=["weak", "nodeshard"])
    ap.add_argument("--method", default="auto")
    ap.add_argument("--tile", default="")
    ap.add_argument("--no-sweep", action="store_true", help="skip the m = 3..8 sweep lines")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline measurement")
    ap.add_argument("--no-graph", action="store_true", help="launch the step kernel by kernel (no CUDA graph)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", FALLBACK_HBM)), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return FALLBACK_HBM, 1965.0, "fallback"


def fp_peak_tflops(fp64, sm_mhz, sms=148):
    """Non-tensor FMA peak derived from unit counts:
    148 SMs x (64 FP64 | 128 FP32 FMA lanes) x 2 flop x clock."""
    lanes = 64 if fp64 else 128
    return sms * lanes * 2 * sm_mhz * 1e6 / 1e12


def algorithmic(w, deg_fp64=True):
    """Per-launch algorithmic bytes and flops:
    resampling: B*c*prod(Ntilde) + B*c*M + r*D*M bytes,
                2*M*[B*2*sum_{d=1..D}(2m)^d + 2m*D*deg] flops (deg = 2m, the paper's);
    deconv/pad: 2*B*c*prod N (the zero padding is written once per plan); crop: 2*B*c*prod N
    (cell mode: the spread rewrites every cell, so no re-zeroing)."""
    c = 16 if w["precision"] == "c128" else 8
    r = 8 if w["precision"] == "c128" else 4
    D, M, B, m = len(w["N"]), w["M"], w["batch"], w["m"]
    nt = int(np.prod([2 * math.ceil(w["sigma"] * n / 2) for n in w["N"]]))
    nn = int(np.prod(w["N"]))
    res_bytes = B * c * nt + B * c * M + r * D * M
    res_flops = 2 * M * (B * 2 * sum((2 * m) ** d for d in range(1, D + 1)) + 2 * m * D * (2 * m))
    return dict(resample_bytes=res_bytes, resample_flops=res_flops, deconv_bytes=2 * B * c * nn,
                crop_bytes=2 * B * c * nn, zero_bytes=B * c * nt, grid_cells=nt)


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


# ----------------------------------------------------------------------------- reference arm

def oracle_step(w, sample_nodes):
    """One oracle step (direct + adjoint NFFT, the same step as our arm's) on
    the first `sample_nodes` nodes; returns nodes processed."""
    from oracle import nfft as onfft
    nodes = w["nodes"][:sample_nodes].astype(np.float64)
    for b in range(w["batch"]):
        onfft.forward(nodes, w["fhat"][b], w["N"], w["m"], w["sigma"])
        onfft.adjoint(nodes, w["f"][b][:sample_nodes], w["N"], w["m"], w["sigma"])
    return sample_nodes * w["batch"]


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def measure_oracle(w, budget_s=12.0, max_reps=None):
    """Times the oracle as it stands on a bounded sample of the workload."""
    t0 = time.perf_counter()
    n = oracle_step(w, w["M"])
    dt = time.perf_counter() - t0
    reps, tot_nodes, tot_t = 1, n, dt
    while tot_t < budget_s and (max_reps is None or reps < max_reps):
        t0 = time.perf_counter()
        tot_nodes += oracle_step(w, w["M"])
        tot_t += time.perf_counter() - t0
        reps += 1
    return dict(value=tot_nodes / tot_t, unit=UNIT, cores=1, kind="oracle",
                sample=f"{reps} full oracle step(s) (direct + adjoint NFFT, fp64 numpy) on the "
                       f"bench workload; numpy FFT/bincount run single-threaded ({cpu_cores()} host cores available)")


def run_reference(a):
    from paper_2208_00049_b200 import workloads
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = workloads.make(a.config, seed=0, m=a.m)
    for _ in range(a.warmup):
        oracle_step(w, w["M"])
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        oracle_step(w, w["M"])
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = a.steps * w["M"] * w["batch"] / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(a, w),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"each step = the full workload through the numpy oracle ({cpu_cores()} cores available)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(a, w, extra=None):
    d = {"workload": f"{a.config}: {len(w['N'])}D N={'x'.join(map(str, w['N']))} M={w['M']} "
                     f"{'ComplexF64' if w['precision'] == 'c128' else 'ComplexF32'} sigma={w['sigma']} m={w['m']} "
                     f"batch={w['batch']}; step = one nfft_execute of the direct + adjoint NFFT on the precomputed "
                     f"plan (independent inputs, adjoint overlaps forward; the node binning/sort is plan setup, timed "
                     f"separately as in SURVEY 8(d): see with_precompute / stages_ms_mean.precompute)",
         "nodes": "uniform i.i.d. in [-1/2,1/2)^D, seed 0", "l2": "flushed before every step (256 MiB write)",
         "parallelism": f"{'nodeshard' if a.mode == 'nodeshard' else 'independent transform per GPU'} x{a.gpus}"}
    if extra:
        d.update(extra)
    return d


# ----------------------------------------------------------------------------- our arm

def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist
    import paper_2208_00049_b200 as pkg
    from paper_2208_00049_b200 import workloads
    from paper_2208_00049_b200.dist import ShardedNfft

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    hbm, sm_max, peak_src = peaks()

    def barrier():
        if world > 1:
            dist.barrier()

    seed = rank if a.mode == "weak" else 0
    w = workloads.make(a.config, seed=seed, m=a.m)
    tile = tuple(int(x) for x in a.tile.split(",")) if a.tile else None

    def build_plan(wk, timing):
        with torch.cuda.stream(stream):
            nodes = torch.from_numpy(wk["nodes"]).to(dev)
            kw = dict(m=wk["m"], sigma=wk["sigma"], precision=wk["precision"], batch=wk["batch"], tile=tile,
                      stream=stream.cuda_stream, device=local, method=a.method, timing=timing, check_nodes=False)
            if a.mode == "nodeshard":
                sp = ShardedNfft(nodes, wk["N"], **kw)
                sp.precompute()
                return sp, sp.plan, nodes
            p = pkg.NfftPlan(nodes, wk["N"], **kw)
            p.precompute()
            return p, p, nodes

    flush_w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)

    class _Flush:
        """L2 flush between steps: write 256 MiB (> 126 MB L2), then read another
        256 MiB so the write-back of the dirty lines also happens here and not
        inside the next timed step."""
        @staticmethod
        def zero_():
            flush_w.zero_()
            flush_sink.copy_(flush_r.sum())
    flush = _Flush()

    def run_steps(wk, steps, warmup, use_graph=not a.no_graph, staged=False, with_pre=False):
        """K timed steps. Default: the step is one nfft_execute of the direct and
        the adjoint NFFT on the precomputed plan (adjoint || forward on plan-
        internal streams), captured as one CUDA graph, timed with CUDA events on
        the plan stream. with_pre=True: the same execute also re-runs the
        precompute (binning + sort, concurrent with the forward deconv + FFT).
        staged=True: the seven stages one after another in ONE graph with
        external event-record nodes between them -> live per-stage (per-kernel)
        durations inside a single graph launch (no per-stage launch gap)."""
        obj, plan, nodes = build_plan(wk, False)
        with torch.cuda.stream(stream):
            fhat = torch.from_numpy(wk["fhat"]).to(dev)
            f = torch.from_numpy(wk["f"]).to(dev)
            fout = torch.zeros((wk["batch"], wk["M"]), dtype=plan.tdtype_c, device=dev)
            yout = torch.empty((wk["batch"],) + tuple(wk["N"]), dtype=plan.tdtype_c, device=dev)
        stream.synchronize()
        shard = a.mode == "nodeshard"
        from paper_2208_00049_b200.dist import allreduce_sum
        names = ["precompute", "deconv", "fft_fwd", "interp", "spread", "fft_adj", "crop"]
        stage_fns = [lambda: plan.run_stage("precompute"), lambda: plan.run_stage("fwd_deconv", fhat),
                     lambda: plan.run_stage("fwd_fft"), lambda: plan.run_stage("fwd_interp", None, fout),
                     lambda: plan.run_stage("adj_spread", f), lambda: plan.run_stage("adj_fft"),
                     lambda: plan.run_stage("adj_crop", None, yout)]
        sev = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(names) + 1)]
               for _ in range(2)] if staged else None

        def one(slot=0):
            if staged:
                for k, fn in enumerate(stage_fns):
                    sev[slot][k].record(stream)
                    fn()
                sev[slot][len(names)].record(stream)
                return
            plan.execute(with_pre, fhat, fout, f, yout)
            if shard:
                allreduce_sum(fout)
                allreduce_sum(yout)

        for _ in range(warmup):
            with torch.cuda.stream(stream):
                flush.zero_()
                one(0)
        stream.synchronize()
        launches_per_step = 0
        g = None
        if use_graph:
            g = torch.cuda.CUDAGraph()
            l0 = plan.launches()
            with torch.cuda.graph(g, stream=stream):
                one(1)
            launches_per_step = plan.launches() - l0
        stream.synchronize()
        l0 = plan.launches()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
        stage = {n: [] for n in names} if staged else {}
        barrier()
        torch.cuda.synchronize(dev)
        with ClockSampler(local) as clk:
            for s in range(steps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                    ev[s][0].record(stream)
                    if g is not None:
                        g.replay()
                    else:
                        one(1)
                    ev[s][1].record(stream)
                if staged:  # the graph's event nodes are reused: read them every step
                    stream.synchronize()
                    for k, n in enumerate(names):
                        stage[n].append(sev[1][k].elapsed_time(sev[1][k + 1]))
            torch.cuda.synchronize(dev)
        barrier()
        launches = launches_per_step * steps if use_graph else plan.launches() - l0
        ms = sum(ev[s][0].elapsed_time(ev[s][1]) for s in range(steps))
        del g
        obj.close()
        return ms, stage, launches, clk.summary()

    ms, _, launches, clocks = run_steps(w, a.steps, a.warmup)
    # the same step with the precompute (binning + sort) re-run inside it
    n_pre = max(20, min(a.steps, 100))
    ms_pre, _, _, _ = run_steps(w, n_pre, a.warmup, with_pre=True)
    # third timed region: the seven stages one after another in one graph, live per-kernel durations
    ms_staged, stage, _, _ = run_steps(w, n_pre, a.warmup, staged=True)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    units_per_rank = w["M"] * w["batch"]
    total_units = units_per_rank * (world if a.mode == "weak" else 1)
    value = total_units * a.steps / (ms_max * 1e-3)

    # roofline of the dominant library kernel (by mean share of the step)
    alg = algorithmic(w)
    means = {k: (statistics.mean(v) if v else 0.0) for k, v in stage.items()}
    # dominant single library kernel (precompute is three kernels; cuFFT is not ours)
    mine = {k: v for k, v in means.items() if k in ("deconv", "interp", "spread", "crop")}
    dom = max(mine, key=mine.get)
    bytes_of = {"interp": alg["resample_bytes"], "spread": alg["resample_bytes"], "deconv": alg["deconv_bytes"],
                "crop": alg["crop_bytes"], "allreduce_fwd": 0, "allreduce_adj": 0,
                "precompute": (8 * len(w["N"]) + 4 * 6) * w["M"]}
    flops_of = {"interp": alg["resample_flops"], "spread": alg["resample_flops"]}
    fp64 = w["precision"] == "c128"
    fp_peak = fp_peak_tflops(fp64, sm_max)
    t_hbm = bytes_of[dom] / (hbm * 1e9)
    t_fp = flops_of.get(dom, 0) / (fp_peak * 1e12)
    dom_s = means[dom] * 1e-3
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{a.config}:m{w['m']}:{dom}")
    if t_fp > t_hbm:
        roof = {"bound": "alu", "achieved": flops_of[dom] / dom_s / 1e12, "peak": fp_peak, "unit": "TFLOP/s",
                "peak_source": f"derived: 148 SM x {'64 FP64' if fp64 else '128 FP32'} FMA x 2 x {sm_max:.0f} MHz"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_of[dom] / dom_s / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)" if peak_src == "measured" else "fallback 6650 GB/s"}
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": traffic, "kernel": dom,
                 "algorithmic_bytes": bytes_of[dom], "algorithmic_flops": flops_of.get(dom, 0),
                 "kernel_ms_mean": means[dom], "kernel_share": means[dom] / (ms_max / a.steps)})

    # end-to-end through the public API with pinned host buffers (rank-local)
    e2e = None
    if not a.no_e2e and a.mode == "weak":
        e2e = measure_e2e(a, w, dev, stream, tile, local, world)

    sweep = None
    if not a.no_sweep and rank == 0 and world == 1 and a.config in ("cfg2_1d_2e18", "cfg3_2d_512"):
        sweep = {}
        for mm in range(3, 9):
            wk = workloads.make(a.config, seed=0, m=mm)
            msk, _, _, _ = run_steps(wk, 20, 3)
            _, st, _, _ = run_steps(wk, 20, 3, staged=True)
            sweep[f"m{mm}"] = {"nodes_per_s": wk["M"] * 20 / (msk * 1e-3),
                               "interp_ms": statistics.mean(st["interp"]), "spread_ms": statistics.mean(st["spread"])}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = measure_oracle(w)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "weak" if a.mode == "weak" else "strong", "vs_baseline": None,
            "dtype": "f64" if fp64 else "f32", "data": "synthetic",
            "config": config_dict(a, w),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "stages_ms_mean": means, "ms_per_step_sequential": ms_staged / n_pre,
            "with_precompute": {"ms_per_step": ms_pre / n_pre,
                                "value": units_per_rank * (world if a.mode == "weak" else 1) / (ms_pre / n_pre * 1e-3),
                                "unit": UNIT, "note": "step + node binning/sort (nfft_precompute) re-run every step"},
            "precompute_nodes_per_s": units_per_rank / w["batch"] / (means["precompute"] * 1e-3),
        }
        if sweep:
            line["m_sweep"] = sweep
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_e2e(a, w, dev, stream, tile, local, world, steps=None):
    """Same metric through the C ABI with pinned HOST buffers: per step one
    nfft_execute of the direct NFFT (host fhat -> host f) and the adjoint
    (host f -> host y) on the precomputed plan; host<->device copies are inside
    the timed region (the final event follows the downloads)."""
    import torch
    import paper_2208_00049_b200 as pkg
    steps = steps or max(5, min(a.steps, 50))

    def pinned(arr):
        t = torch.from_numpy(np.ascontiguousarray(arr)).pin_memory()
        return t, t.numpy()

    _, nodes_h = pinned(w["nodes"])
    _, fhat_h = pinned(w["fhat"])
    _, f_h = pinned(w["f"])
    _, fout_h = pinned(np.empty((w["batch"], w["M"]), w["f"].dtype))
    _, yout_h = pinned(np.empty((w["batch"],) + tuple(w["N"]), w["fhat"].dtype))
    plan = pkg.NfftPlan(nodes_h, w["N"], m=w["m"], sigma=w["sigma"], precision=w["precision"], batch=w["batch"],
                        tile=tile, stream=stream.cuda_stream, device=local, method=a.method, check_nodes=False)

    plan.precompute()

    def step():
        # one nfft_execute with host buffers: the direct NFFT's upload / download run on its own
        # stream, concurrently with the adjoint's (include/nfft.h); outputs are valid after the sync
        plan.execute(False, fhat_h, fout_h, f_h, yout_h)

    for _ in range(3):
        step()
    stream.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    t1.synchronize()
    ms = t0.elapsed_time(t1)
    plan.close()
    h2d = w["fhat"].nbytes + w["f"].nbytes
    d2h = fout_h.nbytes + yout_h.nbytes
    return {"value": w["M"] * w["batch"] * steps / (ms * 1e-3) * world, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps}


if __name__ == "__main__":
    sys.exit(main())
