"""Batch sharding across GPUs.

Checksum groups are independent (reference abft/protected.py:103 keeps no
cross-group state), so a batch shards by contiguous group-aligned slices:
each rank runs the single-GPU protected path on its slice, outputs stay where
they were computed, and the only collective is a reduction of the fault
counters (NCCL all-reduce over NVLink on the B200 box; gloo in the CPU tests)
plus a gather of the (normally empty) flagged / corrected / unrecoverable
records. Group and signal indices are global, like the reference's
``start + idx`` (protected.py:130).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .abft.protected import RunReport, run_protected


def shard_range(batch: int, bs: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) signal range of `rank`: whole groups, balanced within one group."""
    if batch % bs:
        raise ValueError(f"batch size {batch} not divisible by group size {bs}")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    groups = batch // bs
    base, extra = divmod(groups, world)
    g0 = rank * base + min(rank, extra)
    g1 = g0 + base + (1 if rank < extra else 0)
    return g0 * bs, g1 * bs


def _offset(report: RunReport, start: int, bs: int) -> RunReport:
    g0 = start // bs
    report.flagged = [{**f, "group": f["group"] + g0, "signal": f["signal"] + start}
                      for f in report.flagged]
    report.corrected = [{**c, "group": c["group"] + g0, "signal": c["signal"] + start}
                        for c in report.corrected]
    report.unrecoverable = [g + g0 for g in report.unrecoverable]
    return report


def merge_reports(local: RunReport, group=None, device=None) -> RunReport:
    """All-reduce the counters and gather the records of every rank's report."""
    if not dist.is_available() or not dist.is_initialized():
        return local
    dev = device if device is not None else (
        torch.device("cuda", torch.cuda.current_device())
        if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    counts = torch.tensor([local.groups, local.recompute_count, local.pass_count],
                          dtype=torch.int64, device=dev)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    mx = torch.tensor([local.max_rel_discrepancy], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    records = [None] * dist.get_world_size(group)
    dist.all_gather_object(records, (local.flagged, local.corrected, local.unrecoverable),
                           group=group)
    out = RunReport(scheme=local.scheme, delta=local.delta, groups=int(counts[0]))
    for fl, co, un in records:
        out.flagged.extend(fl)
        out.corrected.extend(co)
        out.unrecoverable.extend(un)
    out.flagged.sort(key=lambda f: (f["group"], f["signal"]))
    out.corrected.sort(key=lambda c: (c["group"], c["signal"]))
    out.unrecoverable.sort()
    out.recompute_count = int(counts[1])
    out.pass_count = int(counts[2])
    out.max_rel_discrepancy = float(mx[0])
    return out


def run_protected_sharded(plan, twiddles, local_batch, start: int, scheme="two_sided_group",
                          cfg=None, injector=None, enc=None, inverse=False, group=None):
    """Protected transform of this rank's slice [start, start + len) of a
    global batch; returns (local outputs, global RunReport, local PassCounter).
    A BitFlipInjector's global signal index is translated to the slice."""
    from .fault_lab.bits import BitFlipInjector, FaultSpec

    inj = injector
    if isinstance(injector, BitFlipInjector):
        spec = injector.spec
        inj = BitFlipInjector(FaultSpec(spec.run_id, spec.signal_idx - start, spec.element_idx,
                                        spec.component, spec.bit, spec.stage))
        inj.fired = injector.fired
    out, rep, cnt = run_protected(plan, twiddles, local_batch, scheme, cfg, injector=inj, enc=enc,
                                  inverse=inverse)
    if isinstance(injector, BitFlipInjector) and inj.fired:
        injector.fired = True
    return out, merge_reports(_offset(rep, start, plan.bs), group), cnt
