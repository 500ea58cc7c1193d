"""Benchmark: BASELINE.json configs[1] — FP32 single-kernel FFT sweep
N = 2^3 .. 2^13, a 1 GiB batch per size per GPU, two-sided ABFT on
(two_sided_group), plus ABFT-off and cuFFT (torch.fft) comparisons.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one protected pass of the hot path over every size of the sweep
(11 fused launches, 11 GiB in + 11 GiB out per GPU). Multi-GPU: one process
per GPU (torchrun), each rank owns its own 1 GiB batches (batch sharding, weak
scaling); the only collective is an NCCL all-reduce of the fault counters.
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import ctypes
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

METRIC = "batched FFT GFLOP/s & HBM GB/s (FP32/FP64, ABFT on) vs roofline; ABFT overhead %"
SIZES = list(range(3, 14))            # log2 N
BATCH_BYTES = 1 << 30                 # per size per GPU (complex64 input)
WORKLOAD = ("C2: FP32 single-kernel FFT sweep N=2^3..2^13, 1 GiB complex64 batch per size "
            "per GPU, two-sided ABFT (two_sided_group) on")


def flops(n, batch):
    return 5.0 * n * math.log2(n) * batch


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML every 5 ms while
    the timed region runs (the recipe's nvidia-smi clocks line, in-process).
    NVML is initialised before the timed region and one sample is taken at
    start and at stop, so even a short region has samples."""

    NAMES = {"HwSlowdown": "hw_slowdown", "HwThermalSlowdown": "hw_thermal_slowdown",
             "SwThermalSlowdown": "sw_thermal_slowdown", "SwPowerCap": "sw_power_cap",
             "HwPowerBrakeSlowdown": "hw_power_brake"}

    def __init__(self, index, period=0.005):
        self.index = index
        self.period = period
        self.samples = []
        self.reasons = set()
        self.sm_max = None
        self._stop = threading.Event()
        self._thr = None
        self.err = None
        self._nv = self._h = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self.sm_max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._bits = {getattr(nv, "nvmlClocksEventReason" + k): v for k, v in self.NAMES.items()}
        except Exception as exc:  # pragma: no cover - depends on the box
            self.err = repr(exc)

    def _sample(self):
        nv = self._nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for bit, nm in self._bits.items():
            if r & bit:
                self.reasons.add(nm)

    def _run(self):
        try:
            while not self._stop.wait(self.period):
                self._sample()
        except Exception as exc:  # pragma: no cover
            self.err = repr(exc)

    def start(self):
        if self._nv is None:
            return
        self._sample()
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def stop(self):
        self._stop.set()
        if self._thr is not None:
            self._thr.join(timeout=5)
        if self._nv is not None:
            try:
                self._sample()
            except Exception as exc:  # pragma: no cover
                self.err = repr(exc)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max,
                    "reasons": [self.err or "no samples"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.sm_max,
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


# -------------------------------------------------------------- CPU baseline
def _cpu_shard(args):
    """One worker: the oracle (reference restatement) on a shard of groups."""
    logn, nsig, seed, kernel = args
    sys.path.insert(0, ROOT)
    from oracle import port as P
    n = 1 << logn
    rng = np.random.default_rng([seed, logn])
    x = (rng.standard_normal((nsig, n)) + 1j * rng.standard_normal((nsig, n))).astype(np.complex64)
    plan = P.shrink_bs(P.plan_for(n, "fp32", batch=nsig), nsig)
    tw = P.twiddles_for(plan)
    enc = P.encoding_for("wang", n)
    t0 = time.perf_counter()
    P.protected(plan, tw, x, "two_sided_group", delta=1e-4, enc=enc, kernel=kernel)
    return time.perf_counter() - t0


def cpu_reference(sample_elems=1 << 22, cores=None):
    """Time the reference CPU path (oracle port; the reference's own compiled
    Cython butterfly when oracle/_ref is built) over a bounded sample of the
    sweep: `sample_elems` complex64 samples per size, sharded by checksum
    group over all host cores. Each shard times only its run_protected call;
    the parallel time is the sum of shard times / cores (shards are
    independent, so this is the ideal all-core throughput of the reference).
    Returns (GFLOP/s, cores, sample text, kind)."""
    import multiprocessing as mp
    from oracle import port as P
    kernel = "ref" if P.have_ref_kernel() else "c"
    cores = cores or os.cpu_count() or 1
    jobs = []
    total_flops = 0.0
    for logn in SIZES:
        n = 1 << logn
        nsig = max(16, sample_elems // n)
        per = max(16, (nsig // cores) // 16 * 16)
        shards = max(1, nsig // per)
        for s in range(shards):
            jobs.append((logn, per, s, kernel))
        total_flops += flops(n, per * shards)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        times = pool.map(_cpu_shard, jobs, chunksize=1)
    par = sum(times) / cores
    sample = (f"{sample_elems} complex64 samples per size, N=2^3..2^13 ({len(jobs)} shards), "
              f"run_protected two_sided_group (Wang encoding precomputed), sharded by checksum "
              f"group over {cores} processes, time = sum(shard times)/cores; butterfly kernel: "
              f"{'reference _stockham compiled from /root/reference (oracle/_ref)' if kernel == 'ref' else 'C restatement (oracle/stockham.c)'}")
    return total_flops / par / 1e9, cores, sample, "port"


# ------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2405_02520_b200 import _lib, build_twiddles, make_plan, run_protected
    from paper_2405_02520_b200.abft import DetectionConfig, Scheme, make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    total_elems = BATCH_BYTES // 8
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(total_elems, dtype=torch.complex64, device=dev, generator=g)
    y = torch.empty_like(x)

    cases = []
    for logn in SIZES:
        n = 1 << logn
        b = total_elems // n
        plan = fit_group_size(make_plan(n, "fp32", batch=b), b)
        enc = make_encoding("wang", n)
        row = enc.device_row(torch.complex64, False)
        h = native_plan(plan, local_rank)
        rep = _lib.Report()
        cap = 64
        flags = (_lib.Flag * cap)()
        i64 = (ctypes.c_int64 * cap)
        cg, cs, ur = i64(), i64(), i64()
        rep.flagged, rep.flagged_cap = flags, cap
        rep.corrected_group, rep.corrected_signal, rep.corrected_cap = cg, cs, cap
        rep.unrecoverable, rep.unrecoverable_cap = ur, cap
        cases.append(dict(logn=logn, n=n, b=b, plan=plan, h=h, row=row, rep=rep,
                          keep=(flags, cg, cs, ur)))

    def launch(c, scheme):
        code = _lib.SCHEME_CODE[scheme]
        _lib.check(lib.tfft_protect_launch(c["h"].handle, x.data_ptr(), y.data_ptr(), c["b"], code,
                                           1e-4, 0.0, c["row"].data_ptr(), None, None, 0,
                                           ctypes.byref(c["rep"]), sp), "launch")

    def finish(c, scheme):
        code = _lib.SCHEME_CODE[scheme]
        _lib.check(lib.tfft_protect_finish(c["h"].handle, x.data_ptr(), y.data_ptr(), c["b"], code,
                                           1e-4, 0.0, c["row"].data_ptr(), None, 0,
                                           ctypes.byref(c["rep"]), sp), "finish")

    def step(scheme, events=None):
        for i, c in enumerate(cases):
            if events is not None:
                events[i][0].record(stream)
            launch(c, scheme)
            if events is not None:
                events[i][1].record(stream)
        for c in cases:
            finish(c, scheme)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step("two_sided_group")
    counters = np.zeros(4, dtype=np.int64)
    max_rel = 0.0
    per_n = [[] for _ in cases]
    clocks = ClockSampler(local_rank)
    barrier()
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
            for _ in cases] for _ in range(args.steps)]
    t_start.record(stream)
    for s in range(args.steps):
        step("two_sided_group", evs[s])
        for c in cases:
            r = c["rep"]
            counters += np.array([r.n_flagged, r.n_corrected, r.n_unrecoverable, r.recompute_count])
            max_rel = max(max_rel, r.max_rel_discrepancy)
    t_end.record(stream)
    barrier()
    clk = clocks.stop()
    ms_total = t_start.elapsed_time(t_end)
    for s in range(args.steps):
        for i in range(len(cases)):
            per_n[i].append(evs[s][i][0].elapsed_time(evs[s][i][1]))
    ms_step_local = ms_total / args.steps

    # ---- ABFT off and cuFFT on the same buffers (outside the timed region)
    off_n, cufft_n = [[] for _ in cases], [[] for _ in cases]
    for _ in range(2):
        step("none")
    for s in range(args.steps):
        ev = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
              for _ in cases]
        step("none", ev)
        torch.cuda.synchronize()
        for i in range(len(cases)):
            off_n[i].append(ev[i][0].elapsed_time(ev[i][1]))
    for i, c in enumerate(cases):
        xv = x.view(c["b"], c["n"])
        yv = y.view(c["b"], c["n"])
        torch.fft.fft(xv, out=yv)
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.fft.fft(xv, out=yv)
            e1.record(stream)
            torch.cuda.synchronize()
            cufft_n[i].append(e0.elapsed_time(e1))

    # ---- collectives: max step time over ranks, NCCL-reduced fault counters
    ms_step = ms_step_local
    if world > 1:
        t = torch.tensor([ms_step_local], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        ct = torch.tensor(counters, device=dev)
        dist.all_reduce(ct, op=dist.ReduceOp.SUM)
        counters = ct.cpu().numpy()
        mr = torch.tensor([max_rel], device=dev, dtype=torch.float64)
        dist.all_reduce(mr, op=dist.ReduceOp.MAX)
        max_rel = float(mr.item())

    # ---- e2e: public API, host (pinned) buffers, H2D + D2H inside the timed region
    e2e = None
    if rank == 0 or world > 1:
        xh = x.cpu().pin_memory()
        e2e_steps = max(1, min(args.steps, 3))
        cfg = DetectionConfig(delta=1e-4)
        tws = [build_twiddles(c["plan"]) for c in cases]
        out = None
        for _ in range(2):  # warm exactly like the timed loop (encodings, both pinned output blocks)
            for c, tw in zip(cases, tws):
                out, rep, _ = run_protected(c["plan"], tw, xh.view(c["b"], c["n"]),
                                            Scheme.TWO_SIDED_GROUP, cfg)
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            for c, tw in zip(cases, tws):
                out, rep, _ = run_protected(c["plan"], tw, xh.view(c["b"], c["n"]),
                                            Scheme.TWO_SIDED_GROUP, cfg)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1000 / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        step_flops_all = world * sum(flops(c["n"], c["b"]) for c in cases)
        e2e = {"value": step_flops_all / (e2e_ms / 1000) / 1e9, "unit": "GFLOP/s",
               "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(sum(c["b"] * c["n"] * 8 for c in cases)),
               "d2h_bytes_per_step": int(sum(c["b"] * c["n"] * 8 for c in cases)),
               "api": ("paper_2405_02520_b200.run_protected(pinned host batch -> numpy) -> C-ABI "
                       "tfft_run_protected_host: H2D / fused transform / D2H streamed in 32 MiB "
                       "group-aligned chunks on three streams")}

    if rank != 0:
        return
    hbm, peak_kind = peaks()
    sweep = []
    tot_bytes = tot_on = tot_off = tot_cufft = 0.0
    for i, c in enumerate(cases):
        on = statistics.median(per_n[i])
        off = statistics.median(off_n[i])
        cf = statistics.median(cufft_n[i])
        by = 2.0 * c["b"] * c["n"] * 8
        tot_bytes += by
        tot_on += on
        tot_off += off
        tot_cufft += cf
        sweep.append({"n": c["n"], "batch": c["b"], "ms_abft_on": round(on, 4),
                      "ms_abft_off": round(off, 4), "ms_cufft": round(cf, 4),
                      "gflops_abft_on": round(flops(c["n"], c["b"]) / on / 1e6, 1),
                      "hbm_gbs_abft_on": round(by / on / 1e6, 1),
                      "hbm_frac_abft_on": round(by / on / 1e6 / hbm, 4),
                      "abft_overhead_pct": round(100 * (on / off - 1), 2),
                      "vs_cufft": round(cf / on, 4)})
    step_flops = sum(flops(c["n"], c["b"]) for c in cases) * world
    achieved = tot_bytes / tot_on / 1e6
    # DRAM bytes per launch of these kernels from the committed ncu launch
    # list (tools/launch_summary.py), averaged over the sweep's launches like
    # `achieved` (algorithmic: 2 GiB per launch)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_r01.json")
    if os.path.exists(tpath):
        try:
            by_n = json.load(open(tpath))["dram_bytes_per_launch_by_n"]
            vals = [by_n[str(c["n"])] for c in cases if str(c["n"]) in by_n]
            if len(vals) == len(cases):
                traffic = round(sum(vals) / len(vals))
        except Exception:
            traffic = None
    cpu = None
    if world == 1 and not args.skip_cpu:
        v, cores, sample, kind = cpu_reference()
        cpu = {"value": round(v, 4), "unit": "GFLOP/s", "cores": cores, "kind": kind,
               "sample": sample}
    line = {
        "metric": METRIC,
        "value": round(step_flops / (ms_step / 1000) / 1e9, 1),
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device Philox complex normal), no faults injected",
        "config": {"workload": WORKLOAD, "sizes": [c["n"] for c in cases],
                   "batch_bytes_per_size_per_gpu": BATCH_BYTES, "scheme": "two_sided_group",
                   "delta": 1e-4, "parallelism": f"batch-sharded x{world} (no data collective)",
                   "l2": "inputs (1 GiB per size) larger than L2 (126 MB); no flush needed"},
        "hbm_gbs": round(achieved, 1),
        "abft_overhead_pct": round(100 * (tot_on / tot_off - 1), 2),
        "vs_cufft": round(tot_cufft / tot_on, 4),
        "vs_cufft_abft_off": round(tot_cufft / tot_off, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": traffic, "traffic_algorithmic": 2 * BATCH_BYTES,
                     "kernel": "fft_single_kernel<float, N, ..., ABFT_WANG> (sweep aggregate: "
                               "algorithmic 2*N*8 B per signal / summed event time)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": len(cases) * args.steps,
        "clocks": clk,
        "fault_counters": {"flagged": int(counters[0]), "corrected": int(counters[1]),
                           "unrecoverable": int(counters[2]), "recompute": int(counters[3]),
                           "max_rel_discrepancy": max_rel,
                           "reduced_with": "nccl all_reduce" if world > 1 else "local"},
        "sweep": sweep,
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    if rank != 0:
        return
    ms = []
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        v, cores, sample, kind = cpu_reference(sample_elems=1 << 21)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(v)
            ms.append(dt * 1000)
            info = (cores, sample, kind)
    value = statistics.median(vals)
    cores, sample, kind = info
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.median(ms), 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy default_rng complex normal)",
        "config": {"workload": WORKLOAD, "sizes": [1 << e for e in SIZES],
                   "scheme": "two_sided_group", "delta": 1e-4},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores,
                         "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--skip-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
