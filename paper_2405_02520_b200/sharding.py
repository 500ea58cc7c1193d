"""Batch sharding across GPUs.

Checksum groups are independent (reference abft/protected.py:103 keeps no
cross-group state), so a batch shards by contiguous group-aligned slices:
each rank runs the single-GPU protected path on its slice, outputs stay where
they were computed, and the only collective is a reduction of the fault
counters (NCCL all-reduce over NVLink on the B200 box; gloo in the CPU tests).
The flagged / corrected / unrecoverable records are gathered only when the
reduced counts say some rank has any (normally none). Group and signal
indices are global, like the reference's ``start + idx`` (protected.py:130).

A batch with fewer groups than ranks leaves some ranks an empty slice: they
launch nothing and only join the counter reduction ("replicas only": no
transform is split across GPUs).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .abft.protected import RunReport, run_protected

# all-reduced int64 counters per call (sum): the merged report's scalars,
# the record counts that decide whether records are gathered, and whether the
# fault of a BitFlipInjector fired on some rank
_COUNTS = ("groups", "recompute_count", "pass_count", "n_flagged", "n_corrected", "n_unrecoverable",
           "fired")


def shard_range(batch: int, bs: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) signal range of `rank`: whole groups, balanced within one
    group; empty for surplus ranks when groups < world."""
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


def _reduce_device(group, device):
    if device is not None:
        return device
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def merge_reports(local: RunReport, group=None, device=None, fired: bool = False):
    """Global report of every rank's local one: one all-reduce of the
    counters (sum) and one of the max discrepancy (max); the records are
    all-gathered only when the reduced counts are non-zero. Returns
    (RunReport, fired_on_any_rank)."""
    if not dist.is_available() or not dist.is_initialized():
        return local, fired
    dev = _reduce_device(group, device)
    vals = {"groups": local.groups, "recompute_count": local.recompute_count,
            "pass_count": local.pass_count, "n_flagged": len(local.flagged),
            "n_corrected": len(local.corrected), "n_unrecoverable": len(local.unrecoverable),
            "fired": int(bool(fired))}
    counts = torch.tensor([vals[k] for k in _COUNTS], dtype=torch.int64, device=dev)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    mx = torch.tensor([local.max_rel_discrepancy], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    tot = dict(zip(_COUNTS, counts.tolist()))
    out = RunReport(scheme=local.scheme, delta=local.delta, groups=int(tot["groups"]))
    if tot["n_flagged"] or tot["n_corrected"] or tot["n_unrecoverable"]:
        records = [None] * dist.get_world_size(group)
        dist.all_gather_object(records, (local.flagged, local.corrected, local.unrecoverable),
                               group=group)
        for fl, co, un in records:
            out.flagged.extend(fl)
            out.corrected.extend(co)
            out.unrecoverable.extend(un)
        out.flagged.sort(key=lambda f: (f["group"], f["signal"]))
        out.corrected.sort(key=lambda c: (c["group"], c["signal"]))
        out.unrecoverable.sort()
    out.recompute_count = int(tot["recompute_count"])
    out.pass_count = int(tot["pass_count"])
    out.max_rel_discrepancy = float(mx[0])
    return out, bool(tot["fired"])


def run_protected_sharded(plan, twiddles, local_batch, start: int, scheme="two_sided_group",
                          cfg=None, injector=None, enc=None, inverse=False, group=None):
    """Protected transform of this rank's slice [start, start + len) of a
    global batch; returns (local outputs, global RunReport, local PassCounter).
    `start` must be group-aligned (shard_range gives such slices). A
    BitFlipInjector's global signal index is translated to the slice, and its
    `fired` flag is set on every rank when the fault fired on any of them."""
    from .fault_lab.bits import BitFlipInjector, FaultSpec

    if start < 0 or start % plan.bs:
        raise ValueError(f"slice start {start} is not aligned to the group size {plan.bs}")
    inj = injector
    if isinstance(injector, BitFlipInjector):
        spec = injector.spec
        inj = BitFlipInjector(FaultSpec(spec.run_id, spec.signal_idx - start, spec.element_idx,
                                        spec.component, spec.bit, spec.stage))
        inj.fired = injector.fired
    out, rep, cnt = run_protected(plan, twiddles, local_batch, scheme, cfg, injector=inj, enc=enc,
                                  inverse=inverse)
    fired_here = isinstance(injector, BitFlipInjector) and inj.fired and not injector.fired
    merged, fired_any = merge_reports(_offset(rep, start, plan.bs), group, fired=fired_here)
    if isinstance(injector, BitFlipInjector) and fired_any:
        injector.fired = True
    return out, merged, cnt
