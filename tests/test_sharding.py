"""Batch sharding host logic: group-aligned slices and the report merge over a
world_size-2 gloo process group (CPU; the GPU box runs the same code over
NCCL inside bench.py, and tests/test_gpu_sharding.py runs the whole sharded
protected path on cuda:0 with two gloo ranks)."""

import json
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2405_02520_b200.abft.protected import RunReport
from paper_2405_02520_b200.sharding import _offset, merge_reports, run_protected_sharded, shard_range


def test_shard_range_covers_whole_groups():
    for batch, bs in ((64, 16), (48, 16), (1000, 8), (16, 16), (7, 1), (32, 16), (0, 4)):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(batch, bs, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            assert all(s % bs == 0 and e % bs == 0 for s, e in spans)
            sizes = [(e - s) // bs for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    # fewer groups than ranks: surplus ranks get empty slices (replicas only)
    assert [shard_range(32, 16, 4, r) for r in range(4)] == [(0, 16), (16, 32), (32, 32), (32, 32)]
    with pytest.raises(ValueError):
        shard_range(10, 4, 2, 0)


def test_misaligned_slice_is_rejected():
    from paper_2405_02520_b200.fft_core import make_plan
    plan = make_plan(64, "fp32", batch=16)
    with pytest.raises(ValueError, match="aligned"):
        run_protected_sharded(plan, None, None, start=3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, clean):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bs = 4
    start = rank * 8  # two groups per rank
    local = RunReport(scheme="two_sided_group", delta=1e-4, groups=2)
    local.pass_count = 4
    local.max_rel_discrepancy = 0.5 if rank == 1 else 0.25
    if not clean and rank == 1:
        local.flagged = [{"group": 1, "signal": 5, "discrepancy": 3.0}]
        local.corrected = [{"group": 1, "signal": 5}]
    if not clean and rank == 0:
        local.flagged = [{"group": 0, "signal": 1, "discrepancy": 9.0},
                         {"group": 0, "signal": 2, "discrepancy": 8.0}]
        local.unrecoverable = [0]
    calls = []
    orig = dist.all_gather_object

    def spy(*a, **k):
        calls.append(1)
        return orig(*a, **k)

    dist.all_gather_object = spy
    merged, fired = merge_reports(_offset(local, start, bs), fired=(rank == 1))
    q.put((rank, merged.to_json(), merged.max_rel_discrepancy, fired, len(calls)))
    dist.destroy_process_group()


def _run(clean):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, clean)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_merge_reports_world_size_2_gloo():
    (_, j0, m0, f0, g0), (_, j1, m1, f1, g1) = _run(clean=False)
    assert j0 == j1 and m0 == m1 == 0.5
    assert f0 and f1  # the fault fired on rank 1: every rank's injector learns it
    assert g0 == g1 == 1  # records exist: gathered once
    doc = json.loads(j0)
    assert doc["groups"] == 4 and doc["pass_count"] == 8
    assert [(f["group"], f["signal"]) for f in doc["flagged"]] == [(0, 1), (0, 2), (3, 13)]
    assert doc["corrected"] == [{"group": 3, "signal": 13}]
    assert doc["unrecoverable"] == [0]


def test_clean_merge_skips_the_record_gather():
    (_, j0, m0, _, g0), (_, j1, _, _, g1) = _run(clean=True)
    assert j0 == j1 and g0 == g1 == 0  # counters only: no pickled gather
    doc = json.loads(j0)
    assert doc["groups"] == 4 and doc["flagged"] == [] and doc["pass_count"] == 8
