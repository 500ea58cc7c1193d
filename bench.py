"""Benchmark: BASELINE.json configs[1] (C2) — the FP32 single-kernel FFT sweep
N = 2^3 .. 2^13, a 1 GiB batch per size per GPU, two-sided ABFT on
(two_sided_group) — plus the FP64 multi-pass leg C3 (N = 2^20 .. 2^25, 2 GiB
per GPU), the C5 sweep (FP32 and FP64, N = 2^10 .. 2^25, 1 GiB per size per
GPU: the shape of the 1/2/4/8-GPU scaling runs), ABFT-off and cuFFT
(torch.fft) comparisons, and the reference's CPU path timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--strong] [--skip-cpu] [--skip-c1] [--skip-c3] [--skip-c5]

One step = one protected pass of the hot path over every size of the C2
sweep (11 fused launches, 11 GiB in + 11 GiB out per GPU; every size writes
its own output buffer, so flagged groups are corrected on intact data), then
one NCCL all-reduce of the step's fault counters when N > 1.

Multi-GPU: one process per GPU. Under torchrun the ranks come from the
environment; `--gpus N` without torchrun spawns the N ranks itself
(torch.multiprocessing, NCCL). Weak scaling (default): every rank owns its
own 1 GiB batch per size, i.e. its group-aligned slice of an N GiB global
batch. `--strong`: the global batch per size stays 1 GiB and each rank owns
1/N of it. The e2e leg drives the public sharded API
(`sharding.run_protected_sharded`) with host buffers. Rank 0 prints one JSON
line; times are the max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes
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

METRIC = "batched FFT GFLOP/s & HBM GB/s (FP32/FP64, ABFT on) vs roofline; ABFT overhead %"
SIZES = list(range(3, 14))            # C2: log2 N
C3_SIZES = list(range(20, 26))        # C3: log2 N (fp64, multi-pass)
C5_SIZES = list(range(10, 26))        # C5: log2 N, both precisions (the 1/2/4/8-GPU sweep)
BATCH_BYTES = 1 << 30                 # C2: per size per GPU (complex64 input)
C3_BYTES = 2 << 30                    # C3: per size per GPU (complex128 input)
WORKLOAD = ("C2: FP32 single-kernel FFT sweep N=2^3..2^13, 1 GiB complex64 batch per size "
            "per GPU, two-sided ABFT (two_sided_group) on")


def flops(n, batch):
    return 5.0 * n * math.log2(n) * batch


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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
    """One worker: the oracle (reference restatement with the reference's own
    compiled Cython butterfly) on a shard of checksum groups."""
    logn, nsig, seed, kernel = args
    sys.path.insert(0, ROOT)
    from oracle import port as P
    n = 1 << logn
    rng = np.random.default_rng([seed, logn])
    x = (rng.standard_normal((nsig, n)) + 1j * rng.standard_normal((nsig, n))).astype(np.complex64)
    plan = P.shrink_bs(P.plan_for(n, "fp32", batch=nsig), nsig)
    tw = P.twiddles_for(plan)
    enc = P.encoding_for("wang", n)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):  # one core per worker: no BLAS thread oversubscription
        t0 = time.perf_counter()
        P.protected(plan, tw, x, "two_sided_group", delta=1e-4, enc=enc, kernel=kernel)
        return time.perf_counter() - t0


def _cpu_jobs(sample_elems, shards_per_size):
    jobs, total = [], 0.0
    for logn in SIZES:
        n = 1 << logn
        nsig = max(16, sample_elems // n)
        per = max(16, (nsig // shards_per_size) // 16 * 16)
        k = max(1, nsig // per)
        jobs += [(logn, per, s, None) for s in range(k)]
        total += flops(n, per * k)
    return jobs, total


def cpu_reference(cores=None, single_elems=1 << 24, multi_elems=1 << 25):
    """The reference's CPU path (oracle port; butterflies by the reference's
    own compiled `_stockham` when oracle/_ref is built) over bounded samples
    of the C2 sweep, measured two ways:
      * 1 core: one process, `single_elems` complex64 samples per size, the
        summed run_protected time (the reference as shipped is single-threaded;
        BLAS is held to one thread, threadpoolctl);
      * all cores: `multi_elems` samples per size sharded by checksum group over
        a pool of `cores` processes, timed as the WALL time of the pool map
        (workers warmed first; the wall includes each shard's seeded input draw).
    Returns a dict with both GFLOP/s figures."""
    import multiprocessing as mp
    from oracle import port as P
    kernel = "ref" if P.have_ref_kernel() else "c"
    cores = cores or os.cpu_count() or 1
    jobs1, fl1 = _cpu_jobs(single_elems, 1)
    jobs1 = [(a, b, c, kernel) for a, b, c, _ in jobs1]
    t1 = sum(_cpu_shard(j) for j in jobs1)
    jobsn, fln = _cpu_jobs(multi_elems, cores)
    jobsn = [(a, b, c, kernel) for a, b, c, _ in jobsn]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_shard, [(3, 16, 0, kernel)] * cores)  # warm the workers (imports, kernel load)
        w0 = time.perf_counter()
        shard_t = pool.map(_cpu_shard, jobsn, chunksize=1)
        wall = time.perf_counter() - w0
    butterfly = ("reference _stockham compiled from /root/reference (oracle/_ref)" if kernel == "ref"
                 else "C restatement (oracle/stockham.c)")
    return {
        "one_core_gflops": fl1 / t1 / 1e9, "one_core_s": t1,
        "all_core_gflops": fln / wall / 1e9, "all_core_wall_s": wall,
        "all_core_busy_s": sum(shard_t), "cores": cores, "kind": "port",
        "sample": (f"C2 sweep N=2^3..2^13, run_protected two_sided_group (Wang encoding "
                   f"precomputed); 1 core (input draw outside the clock): {single_elems} complex64 "
                   f"samples per size in one process; all cores: {multi_elems} samples per size in "
                   f"{len(jobsn)} group-aligned shards over {cores} processes, pool wall time incl. each shard's input draw; "
                   f"butterfly: {butterfly}"),
    }


# ------------------------------------------------------------------- ours
class Report:
    """ctypes report buffers for the launch / finish C ABI."""

    def __init__(self, lib_mod, cap=64):
        self.rep = lib_mod.Report()
        self.keep = ((lib_mod.Flag * cap)(), (ctypes.c_int64 * cap)(), (ctypes.c_int64 * cap)(),
                     (ctypes.c_int64 * cap)())
        flags, cg, cs, ur = self.keep
        self.rep.flagged, self.rep.flagged_cap = flags, cap
        self.rep.corrected_group, self.rep.corrected_signal, self.rep.corrected_cap = cg, cs, cap
        self.rep.unrecoverable, self.rep.unrecoverable_cap = ur, cap


def _cases(prec, sizes, per_rank_bytes, device, dev_index):
    import torch

    from paper_2405_02520_b200 import _lib, make_plan
    from paper_2405_02520_b200.abft import make_encoding
    from paper_2405_02520_b200.fft_core import fit_group_size
    from paper_2405_02520_b200.fft_core.plan import native_plan
    esz = 8 if prec == "fp32" else 16
    td = torch.complex64 if prec == "fp32" else torch.complex128
    out = []
    for logn in sizes:
        n = 1 << logn
        b = per_rank_bytes // (esz * n)
        plan = fit_group_size(make_plan(n, prec, batch=b), b)
        enc = make_encoding("wang", n)
        h = native_plan(plan, dev_index)
        out.append(dict(logn=logn, n=n, b=b, plan=plan, h=h, row=enc.device_row(td, False),
                        y=torch.empty((b, n), dtype=td, device=device), esz=esz,
                        passes=_lib.load().tfft_plan_exec_passes(h.handle), rep=Report(_lib)))
    return out


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2405_02520_b200 import _lib, build_twiddles
    from paper_2405_02520_b200.abft import DetectionConfig, Scheme
    from paper_2405_02520_b200.sharding import run_protected_sharded

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    share = world if args.strong else 1
    c2_bytes = BATCH_BYTES // share
    x = torch.randn(c2_bytes // 8, dtype=torch.complex64, device=dev,
                    generator=torch.Generator(device=dev).manual_seed(1234 + rank))
    cases = _cases("fp32", SIZES, c2_bytes, dev, local_rank)

    def launch(c, xx, scheme, delta):
        code = _lib.SCHEME_CODE[scheme]
        _lib.check(lib.tfft_protect_launch(c["h"].handle, xx.data_ptr(), c["y"].data_ptr(), c["b"], code,
                                           delta, 0.0, c["row"].data_ptr(), None, None, 0,
                                           ctypes.byref(c["rep"].rep), sp), "launch")

    def finish(c, xx, scheme, delta):
        code = _lib.SCHEME_CODE[scheme]
        _lib.check(lib.tfft_protect_finish(c["h"].handle, xx.data_ptr(), c["y"].data_ptr(), c["b"], code,
                                           delta, 0.0, c["row"].data_ptr(), None, 0,
                                           ctypes.byref(c["rep"].rep), sp), "finish")

    def step(cs, xx, scheme, delta, events=None):
        """One protected pass over every size: all launches queue first, then
        the per-size detection summaries are read (and rare flags handled)."""
        for i, c in enumerate(cs):
            if events is not None:
                events[i][0].record(stream)
            launch(c, xx, scheme, delta)
            if events is not None:
                events[i][1].record(stream)
        cnt = np.zeros(4, dtype=np.int64)
        mx = 0.0
        if scheme != "none":
            for c in cs:
                finish(c, xx, scheme, delta)
                r = c["rep"].rep
                cnt += np.array([r.n_flagged, r.n_corrected, r.n_unrecoverable, r.recompute_count])
                mx = max(mx, r.max_rel_discrepancy)
        return cnt, mx

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce_counts(cnt, mx):
        """The protected path's one collective: sum of the fault counters
        (and max of the max discrepancy) over the ranks."""
        if world == 1:
            return cnt, mx
        t = torch.tensor(list(cnt) + [0], dtype=torch.float64, device=dev)
        t[-1] = mx
        ct = t[:-1].clone()
        dist.all_reduce(ct, op=dist.ReduceOp.SUM)
        m = t[-1:].clone()
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        return ct.cpu().numpy().astype(np.int64), float(m.item())

    def timed(cs, xx, scheme, delta, steps):
        counters = np.zeros(4, dtype=np.int64)
        max_rel = 0.0
        per = [[] for _ in cs]
        clocks = ClockSampler(local_rank)
        barrier()
        l0 = _lib.launch_count()
        clocks.start()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                for _ in cs] for _ in range(steps)]
        t0.record(stream)
        for s in range(steps):
            cnt, mx = step(cs, xx, scheme, delta, evs[s])
            cnt, mx = reduce_counts(cnt, mx)
            counters += cnt
            max_rel = max(max_rel, mx)
        t1.record(stream)
        barrier()
        clk = clocks.stop()
        launches = _lib.launch_count() - l0
        for s in range(steps):
            for i in range(len(cs)):
                per[i].append(evs[s][i][0].elapsed_time(evs[s][i][1]))
        ms_local = t0.elapsed_time(t1) / steps
        return ms_local, per, counters, max_rel, clk, launches

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def off_and_cufft(cs, xx, reps):
        off, cuf = [[] for _ in cs], [[] for _ in cs]
        step(cs, xx, "none", 1.0)
        for _ in range(reps):
            ev = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in cs]
            step(cs, xx, "none", 1.0, ev)
            torch.cuda.synchronize()
            for i in range(len(cs)):
                off[i].append(ev[i][0].elapsed_time(ev[i][1]))
        for i, c in enumerate(cs):
            xv = xx[:c["b"] * c["n"]].view(c["b"], c["n"])
            torch.fft.fft(xv, out=c["y"])
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                torch.fft.fft(xv, out=c["y"])
                e1.record(stream)
                torch.cuda.synchronize()
                cuf[i].append(e0.elapsed_time(e1))
        return off, cuf

    # ---------------------------------------------------------------- C2
    for _ in range(args.warmup):
        step(cases, x, "two_sided_group", 1e-4)
    ms_local, per_n, counters, max_rel, clk, launches = timed(cases, x, "two_sided_group", 1e-4, args.steps)
    ms_step = max_over_ranks(ms_local)
    off_n, cufft_n = off_and_cufft(cases, x, max(3, min(args.steps, 10)))

    # ---------------------------------------------------------------- e2e
    # the public API with host (pinned) buffers: H2D and D2H inside the timed
    # region; at N > 1 through sharding.run_protected_sharded (global batch =
    # the ranks' slices, start = rank's offset), counters reduced over NCCL
    xh = x.cpu().pin_memory()
    cfg = DetectionConfig(delta=1e-4)
    tws = [build_twiddles(c["plan"]) for c in cases]

    def api_step():
        for c, tw in zip(cases, tws):
            xv = xh[:c["b"] * c["n"]].view(c["b"], c["n"])
            out, rep, _ = run_protected_sharded(c["plan"], tw, xv, rank * c["b"], Scheme.TWO_SIDED_GROUP,
                                                cfg)
        return out

    for _ in range(2):  # warm exactly like the timed loop (encodings, pinned output blocks)
        api_step()
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        api_step()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks((time.perf_counter() - w0) * 1000 / e2e_steps)
    step_flops_all = world * sum(flops(c["n"], c["b"]) for c in cases)
    e2e = {"value": round(step_flops_all / (e2e_ms / 1000) / 1e9, 1), "unit": "GFLOP/s",
           "ms_per_step": round(e2e_ms, 3),
           "h2d_bytes_per_step": int(sum(c["b"] * c["n"] * 8 for c in cases)),
           "d2h_bytes_per_step": int(sum(c["b"] * c["n"] * 8 for c in cases)),
           "api": ("paper_2405_02520_b200.sharding.run_protected_sharded(pinned host slice -> numpy) "
                   "-> run_protected -> C-ABI tfft_run_protected_host (H2D / fused transform / D2H "
                   "streamed in 32 MiB group-aligned chunks on three streams) + NCCL counter reduce"
                   if world > 1 else
                   "paper_2405_02520_b200.run_protected(pinned host batch -> numpy) via "
                   "sharding.run_protected_sharded (world 1) -> C-ABI tfft_run_protected_host: H2D / "
                   "fused transform / D2H streamed in 32 MiB group-aligned chunks on three streams")}
    del xh

    # ---------------------------------------------------------------- C1
    # BASELINE configs[0] (the reference's own CPU-runnable case): FP32
    # N = 1024, batch 256, two-sided, no faults — a 4 MiB latency case: per
    # call wall time of the public run_protected (device tensors; numpy in /
    # out) and the fused launch alone (events), medians of 200 calls
    c1 = None
    if not args.skip_c1:
        from paper_2405_02520_b200 import make_plan, run_protected
        from paper_2405_02520_b200.abft import make_encoding
        from paper_2405_02520_b200.fft_core import fit_group_size
        from paper_2405_02520_b200.fft_core.plan import native_plan
        n1, b1 = 1024, 256
        x1 = np.random.default_rng(rank).standard_normal((b1, 2 * n1)).view(np.complex128).astype(np.complex64)
        plan1 = fit_group_size(make_plan(n1, "fp32", batch=b1), b1)
        tw1 = build_twiddles(plan1)
        xd1 = torch.from_numpy(x1).to(dev)
        clk1 = ClockSampler(local_rank)
        c1 = {"workload": "C1: FP32 N=1024 batch=256 two_sided_group, no faults (4 MiB, fits L2: latency)"}
        clk1.start()
        for name, inp in (("device_api_us", xd1), ("numpy_api_us", x1)):
            for _ in range(20):
                run_protected(plan1, tw1, inp, Scheme.TWO_SIDED_GROUP, cfg)
            ts = []
            for _ in range(200):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                run_protected(plan1, tw1, inp, Scheme.TWO_SIDED_GROUP, cfg)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t0) * 1e6)
            c1[name] = round(statistics.median(ts), 1)
        h1 = native_plan(plan1, local_rank)
        row1 = make_encoding("wang", n1).device_row(torch.complex64)
        y1 = torch.empty_like(xd1)
        rep1 = Report(_lib).rep
        ts = []
        for i in range(220):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.check(lib.tfft_protect_launch(h1.handle, xd1.data_ptr(), y1.data_ptr(), b1, 3, 1e-4, 0.0,
                                               row1.data_ptr(), None, None, 0, ctypes.byref(rep1), sp), "c1")
            e1.record(stream)
            torch.cuda.synchronize()
            _lib.check(lib.tfft_protect_finish(h1.handle, xd1.data_ptr(), y1.data_ptr(), b1, 3, 1e-4, 0.0,
                                               row1.data_ptr(), None, 0, ctypes.byref(rep1), sp), "c1")
            if i >= 20:
                ts.append(e0.elapsed_time(e1) * 1e3)
        c1["fused_launch_us"] = round(statistics.median(ts), 1)
        c1["clocks"] = clk1.stop()
        c1["gflops_device_api"] = round(flops(n1, b1) / (c1["device_api_us"] * 1e-6) / 1e9, 1)
        del xd1, y1

    # ---------------------------------------------------------------- C3
    c3 = None
    if not args.skip_c3:
        for c in cases:
            del c["y"]
        del x
        torch.cuda.empty_cache()
        c3_bytes = C3_BYTES // share
        x3 = torch.randn(c3_bytes // 16, dtype=torch.complex128, device=dev,
                         generator=torch.Generator(device=dev).manual_seed(4321 + rank))
        cases3 = _cases("fp64", C3_SIZES, c3_bytes, dev, local_rank)
        for _ in range(max(2, args.warmup)):
            step(cases3, x3, "two_sided_group", 1e-9)
        steps3 = max(3, min(args.steps, 10))
        ms3, per3, cnt3, mx3, clk3, launches3 = timed(cases3, x3, "two_sided_group", 1e-9, steps3)
        ms3 = max_over_ranks(ms3)
        off3, cuf3 = off_and_cufft(cases3, x3, 3)
        c3 = dict(cases=cases3, per=per3, off=off3, cuf=cuf3, ms=ms3, cnt=cnt3, mx=mx3, clk=clk3,
                  launches=launches3, steps=steps3)
        del x3

    # ---------------------------------------------------------------- C5
    # BASELINE configs[4]: the batch-sharded FP32 / FP64 sweep N = 2^10..2^25,
    # 1 GiB per size per GPU (weak; --strong: 1 GiB per size in total),
    # two-sided ABFT on; time = max over ranks
    c5 = None
    if not args.skip_c5:
        if args.skip_c3:
            for c in cases:
                c.pop("y", None)
            x = None
        torch.cuda.empty_cache()
        c5 = {}
        for prec in ("fp32", "fp64"):
            esz = 8 if prec == "fp32" else 16
            td = torch.complex64 if prec == "fp32" else torch.complex128
            c5_bytes = BATCH_BYTES // share
            x5 = torch.randn(c5_bytes // esz, dtype=td, device=dev,
                             generator=torch.Generator(device=dev).manual_seed(5555 + rank))
            cases5 = _cases(prec, C5_SIZES, c5_bytes, dev, local_rank)
            d5 = 1e-4 if prec == "fp32" else 1e-9
            for _ in range(2):
                step(cases5, x5, "two_sided_group", d5)
            ms5, per5, cnt5, mx5, clk5, l5 = timed(cases5, x5, "two_sided_group", d5, 3)
            c5[prec] = dict(cases=cases5, per=per5, ms=max_over_ranks(ms5), clk=clk5, cnt=cnt5, launches=l5)
            for c in cases5:
                c.pop("y", None)
            del x5
            torch.cuda.empty_cache()

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
    for tname in ("traffic_r02.json", "traffic_r01.json"):
        tpath = os.path.join(ROOT, "profiles", tname)
        if traffic is None and os.path.exists(tpath):
            try:
                by_n = json.load(open(tpath))["dram_bytes_per_launch_by_n"]
                vals = [by_n[str(c["n"])] for c in cases if str(c["n"]) in by_n]
                if len(vals) == len(cases):
                    traffic = round(sum(vals) / len(vals))
            except Exception:
                traffic = None
    cpu = None
    if world == 1 and not args.skip_cpu:
        cr = cpu_reference()
        cpu = {"value": round(cr["all_core_gflops"], 4), "unit": "GFLOP/s", "cores": cr["cores"],
               "kind": cr["kind"], "sample": cr["sample"],
               "one_core": {"value": round(cr["one_core_gflops"], 4), "unit": "GFLOP/s", "cores": 1,
                            "seconds": round(cr["one_core_s"], 2)},
               "all_core_wall_s": round(cr["all_core_wall_s"], 2),
               "all_core_busy_s": round(cr["all_core_busy_s"], 2)}
    c3_out = None
    if c3 is not None:
        rows = []
        t_on = t_off = t_cf = by_exec = by_min = 0.0
        for i, c in enumerate(c3["cases"]):
            on = statistics.median(c3["per"][i])
            off = statistics.median(c3["off"][i])
            cf = statistics.median(c3["cuf"][i])
            per_pass = 2.0 * c["b"] * c["n"] * 16
            t_on += on
            t_off += off
            t_cf += cf
            by_exec += c["passes"] * per_pass
            by_min += 2 * per_pass
            rows.append({"n": c["n"], "batch": c["b"], "passes": c["passes"], "ms_abft_on": round(on, 4),
                         "ms_abft_off": round(off, 4), "ms_cufft": round(cf, 4),
                         "gflops_abft_on": round(flops(c["n"], c["b"]) / on / 1e6, 1),
                         "hbm_gbs_per_executed_pass": round(c["passes"] * per_pass / on / 1e6, 1),
                         "frac_per_executed_pass": round(c["passes"] * per_pass / on / 1e6 / hbm, 4),
                         "frac_vs_2pass_minimum": round(2 * per_pass / on / 1e6 / hbm, 4),
                         "abft_overhead_pct": round(100 * (on / off - 1), 2),
                         "vs_cufft": round(cf / on, 4)})
        c3_out = {
            "workload": ("C3: FP64 multi-pass FFT N=2^20..2^25, 2 GiB complex128 batch per size per GPU, "
                         "two_sided_group ABFT on (delta 1e-9)"),
            "steps": c3["steps"], "ms_per_step": round(c3["ms"], 4),
            "value": round(world * sum(flops(c["n"], c["b"]) for c in c3["cases"]) / (c3["ms"] / 1000) / 1e9, 1),
            "unit": "GFLOP/s", "dtype": "f64",
            "roofline": {"bound": "hbm", "achieved": round(by_exec / t_on / 1e6, 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(by_exec / t_on / 1e6 / hbm, 4),
                         "frac_vs_2pass_minimum": round(by_min / t_on / 1e6 / hbm, 4),
                         "kernel": "fft_pass_kernel<double, L, ...> passes actually launched (+ finalize)"},
            "abft_overhead_pct": round(100 * (t_on / t_off - 1), 2), "vs_cufft": round(t_cf / t_on, 4),
            "gpu_launches": int(c3["launches"]), "clocks": c3["clk"],
            "fault_counters": {"flagged": int(c3["cnt"][0]), "corrected": int(c3["cnt"][1]),
                               "unrecoverable": int(c3["cnt"][2]), "max_rel_discrepancy": c3["mx"]},
            "sweep": rows,
        }
    c5_out = None
    if c5 is not None:
        c5_out = {"workload": ("C5: batch-sharded FP32/FP64 sweep N=2^10..2^25, "
                               f"{'1 GiB in total' if args.strong else '1 GiB per GPU'} per size, "
                               "two_sided_group ABFT on; time = max over ranks"), "unit": "GFLOP/s"}
        for prec, r in c5.items():
            esz = 8 if prec == "fp32" else 16
            rows = []
            for i, c in enumerate(r["cases"]):
                on = statistics.median(r["per"][i])
                per_pass = 2.0 * c["b"] * c["n"] * esz
                rows.append({"n": c["n"], "batch": c["b"], "passes": c["passes"], "ms": round(on, 4),
                             "gflops": round(flops(c["n"], c["b"]) / on / 1e6, 1),
                             "frac_per_executed_pass": round(c["passes"] * per_pass / on / 1e6 / hbm, 4)})
            c5_out[prec] = {
                "value": round(world * sum(flops(c["n"], c["b"]) for c in r["cases"]) / (r["ms"] / 1000) / 1e9, 1),
                "ms_per_step": round(r["ms"], 4), "steps": 3, "gpu_launches": int(r["launches"]),
                "clocks": r["clk"], "flagged": int(r["cnt"][0]), "sizes": rows}
    line = {
        "metric": METRIC,
        "value": round(step_flops / (ms_step / 1000) / 1e9, 1),
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device Philox complex normal), no faults injected",
        "config": {"workload": WORKLOAD, "sizes": [c["n"] for c in cases],
                   "batch_bytes_per_size_per_gpu": c2_bytes, "scheme": "two_sided_group",
                   "delta": 1e-4, "parallelism": f"batch-sharded x{world} (NCCL counter all-reduce only)",
                   "l2": "inputs (1 GiB per size) larger than L2 (126 MB); no flush needed"},
        "hbm_gbs": round(achieved, 1),
        "host_gap_ms_per_step": round(ms_step - tot_on, 4),
        "abft_overhead_pct": round(100 * (tot_on / tot_off - 1), 2),
        "vs_cufft": round(tot_cufft / tot_on, 4),
        "vs_cufft_abft_off": round(tot_cufft / tot_off, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": traffic, "traffic_algorithmic": 2 * c2_bytes,
                     "kernel": "fft_single_kernel<float, N, ..., ABFT_WANG> (sweep aggregate: "
                               "algorithmic 2*N*8 B per signal / summed event time)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "fault_counters": {"flagged": int(counters[0]), "corrected": int(counters[1]),
                           "unrecoverable": int(counters[2]), "recompute": int(counters[3]),
                           "max_rel_discrepancy": max_rel,
                           "reduced_with": "nccl all_reduce per step" if world > 1 else "local"},
        "sweep": sweep,
        "c1": c1,
        "c3": c3_out,
        "c5": c5_out,
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path (the
    oracle port with the reference's compiled butterfly) on all host cores,
    rank 0 only; each step = one all-core wall-timed sample of the C2 sweep."""
    if rank != 0:
        return
    import multiprocessing as mp
    from oracle import port as P
    kernel = "ref" if P.have_ref_kernel() else "c"
    cores = os.cpu_count() or 1
    jobs, fl = _cpu_jobs(1 << 22, cores)
    jobs = [(a, b, c, kernel) for a, b, c, _ in jobs]
    ms, vals = [], []
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_cpu_shard, [(3, 16, 0, kernel)] * cores)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_cpu_shard, jobs, chunksize=1)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                vals.append(fl / dt / 1e9)
                ms.append(dt * 1000)
    value = statistics.median(vals)
    sample = (f"C2 sweep N=2^3..2^13, 4194304 complex64 samples per size, run_protected "
              f"two_sided_group, {len(jobs)} group-aligned shards over {cores} processes, pool wall "
              f"time per step; butterfly: "
              f"{'reference _stockham compiled from /root/reference (oracle/_ref)' if kernel == 'ref' else 'C restatement'}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.median(ms), 2), "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy default_rng complex normal)",
        "config": {"workload": WORKLOAD, "sizes": [1 << e for e in SIZES],
                   "scheme": "two_sided_group", "delta": 1e-4},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _rank_main(rank, world, port, args):
    """Entry of a self-spawned rank (bench.py --gpus N without torchrun)."""
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    _run(args, rank, world, rank)


def _run(args, rank, world, local_rank):
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--strong", action="store_true", help="fixed global batch (1 GiB per size) split over the ranks")
    ap.add_argument("--skip-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--skip-c3", action="store_true", help="skip the FP64 C3 leg")
    ap.add_argument("--skip-c5", action="store_true", help="skip the C5 FP32/FP64 2^10..2^25 sweep")
    ap.add_argument("--skip-c1", action="store_true", help="skip the C1 latency leg")
    args = ap.parse_args()
    if "WORLD_SIZE" in os.environ:  # torchrun
        _run(args, int(os.environ.get("RANK", "0")), int(os.environ["WORLD_SIZE"]),
             int(os.environ.get("LOCAL_RANK", "0")))
        return
    if args.gpus > 1 and args.impl == "ours":
        import socket

        import torch.multiprocessing as mp
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        mp.spawn(_rank_main, args=(args.gpus, port, args), nprocs=args.gpus, join=True)
        return
    _run(args, 0, 1, 0)


if __name__ == "__main__":
    main()
