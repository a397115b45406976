"""Workers, shards and the host-array pipeline on the GPU.

* ``run`` / ``degree_counts`` with ``workers`` (driver.py:210-270): RunStats
  follow the reference's plan (the reference's own test_run_stats and
  test_run_multiworker_stats_cover_all_batches, tests/test_driver.py:129-147),
  and every result is independent of workers and batch size.
* ``parba_multi_run_shards``: one histogram per distinct device, summed by
  NCCL (forced here on one GPU with PARBA_MULTI_NCCL=1; a 2-GPU box also runs
  the two-device case).
* ``generate_block`` into a host array through the native pipeline (u32
  targets over PCIe, rows filled by host threads) vs the 16-byte-row path
  and the oracle.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import pytest

import oracle as O
from conftest import TRIANGLE, ring_edges

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_1602_07106_b200")

UNIFORM = pb.GenParams(n=40, d=3, n0=3, seed_edges=TRIANGLE)  # m0=3, m=114 (reference test_driver.py:24)


def _op(p):
    return O.OParams(n=p.n, d=p.d, n0=p.n0, seed_edges=tuple(int(x) for x in p.seed_edges))


def test_run_stats():
    """Reference tests/test_driver.py:129-138, verbatim expectations."""
    result, stats = pb.run(UNIFORM, pb.DiscardConsumer(), workers=1, batch_size=10)
    assert result == UNIFORM.m - UNIFORM.m0 == 111
    assert stats.edges_emitted == 111
    assert stats.hash_probes > 0
    assert stats.elapsed > 0
    assert len(stats.per_worker) == 1
    ws = stats.per_worker[0]
    assert ws.batches == len(pb.plan_batches(UNIFORM, 10)) == 12
    assert ws.edges == 111


def test_run_multiworker_stats_cover_all_batches():
    """Reference tests/test_driver.py:141-147."""
    result, stats = pb.run(UNIFORM, pb.DiscardConsumer(), workers=3, batch_size=10)
    assert result == 111
    assert len(stats.per_worker) == 3
    assert sum(ws.batches for ws in stats.per_worker) == 12
    assert sum(ws.edges for ws in stats.per_worker) == 111
    assert [ws.worker_id for ws in stats.per_worker] == [0, 1, 2]
    _, one = pb.run(UNIFORM, pb.DiscardConsumer(), workers=1, batch_size=10)
    assert stats.hash_probes == one.hash_probes


def test_run_matches_oracle_across_schedules():
    """Reference tests/test_driver.py:111-118: Collect over workers x batch sizes."""
    p = pb.GenParams(n=800, d=2, n0=3, seed_edges=TRIANGLE)
    want, wp = O.generate_block(_op(p), p.m0, p.m)
    for workers in (1, 2, 4):
        for batch_size in (64, 1 << 16):
            got, stats = pb.run(p, pb.CollectConsumer(), workers=workers, batch_size=batch_size)
            assert np.array_equal(got, want)
            assert stats.edges_emitted == p.m - p.m0 and stats.hash_probes == wp
            assert len(stats.per_worker) == workers
            assert sum(w.batches for w in stats.per_worker) == len(pb.plan_batches(p, batch_size))


@pytest.mark.parametrize("workers", [1, 2, 3, 8])
def test_degree_counts_independent_of_workers(workers):
    p = pb.GenParams(n=30000, d=7, n0=10, seed_edges=ring_edges(10))
    base, bst = pb.degree_counts(p, K=5000, workers=1, batch_size=4096)
    got, st = pb.degree_counts(p, K=5000, workers=workers, batch_size=4096)
    assert np.array_equal(got.counts, base.counts)
    assert st.hash_probes == bst.hash_probes
    assert len(st.per_worker) == workers
    assert sum(w.edges for w in st.per_worker) == p.m - p.m0
    full, _ = pb.degree_counts(p, workers=workers, batch_size=1000)
    ref = np.zeros(p.n, dtype=np.int64)
    blk, _ = O.generate_block(_op(p), p.m0, p.m)
    O.count_block(ref, blk)
    O.count_block(ref, p.seed_edges)
    assert np.array_equal(full.counts, ref)


def test_degree_counts_workers_flags_and_degree_sequences():
    rng = np.random.default_rng(7)
    deg = rng.integers(0, 9, size=4000).astype(np.uint64)
    for kw in (dict(degrees=deg), dict(degrees=deg, no_self_loops=True), dict(d=5, no_parallel_edges=True)):
        p = pb.GenParams(n=4010, n0=10, seed_edges=ring_edges(10), **kw)
        a, sa = pb.degree_counts(p, K=1000, workers=1, batch_size=3000)
        b, sb = pb.degree_counts(p, K=1000, workers=3, batch_size=3000)
        assert np.array_equal(a.counts, b.counts) and sa.hash_probes == sb.hash_probes
        assert sum(w.batches for w in sb.per_worker) == len(pb.plan_batches(p, 3000))


def test_empty_degree_sequence():
    """A degree sequence of zeros generates no edges (m == m0): zero counts,
    no batches, like the reference -- no rank directory needed."""
    p = pb.GenParams(n=8, degrees=np.zeros(8, dtype=np.uint64))
    assert p.m == 0
    counter, st = pb.degree_counts(p)
    assert counter.counts.tolist() == [0] * 8 and st.edges_emitted == 0
    res, st = pb.run(p, pb.DiscardConsumer(), workers=2)
    assert res == 0 and len(st.per_worker) == 2 and sum(w.batches for w in st.per_worker) == 0
    q = pb.GenParams(n=13, n0=10, seed_edges=ring_edges(10), degrees=np.zeros(3, dtype=np.uint64))
    c, _ = pb.degree_counts(q)
    assert c.counts.tolist() == [2] * 10 + [0] * 3


def test_file_writer_workers(tmp_path):
    p = pb.GenParams(n=50000, d=4, n0=3, seed_edges=TRIANGLE)
    want, _ = O.generate_block(_op(p), p.m0, p.m)
    for workers in (1, 3):
        path = str(tmp_path / f"e{workers}.bin")
        with pb.EdgeFileWriter(path, p.m0, p.m - p.m0) as w:
            nbytes, st = pb.run(p, w, workers=workers, batch_size=10_000)
        assert nbytes == 16 * (p.m - p.m0) and len(st.per_worker) == workers
        assert np.array_equal(np.fromfile(path, dtype="<u8").reshape(-1, 2), want)


def test_multi_run_shards_nccl_path(monkeypatch):
    """The NCCL reduce of parba_multi_run_shards, forced on one device."""
    monkeypatch.setenv("PARBA_MULTI_NCCL", "1")
    p = pb.GenParams(n=200_000, d=6, n0=3, seed_edges=TRIANGLE)
    ref = np.zeros(p.n, dtype=np.int64)
    blk, wp = O.generate_block(_op(p), p.m0, p.m)
    O.count_block(ref, blk)
    got, pr, secs = pb.parallel.multi_run(p, [0], mode="full")
    assert np.array_equal(got, ref) and pr == wp and secs > 0
    got, pr, _ = pb.parallel.multi_run(p, [0, 0, 0], mode="window", K=12345)
    assert np.array_equal(got, ref[:12345]) and pr == wp
    ranges = [(p.m0, 1000), (1000, 1000), (1000, 777_777), (777_777, p.m)]
    res, prs = pb.parallel.run_shards(p, "window", 999, ranges, [0] * 4)
    assert np.array_equal(res, ref[:999]) and sum(prs) == wp and prs[1] == 0


# --------------------------------------------------------------------------- owner-routed full histogram


def _routed_full(p, ranges, owners, dev="cuda:0"):
    """Counts of the ranges through parba_degree_full_routed into `owners`
    separately allocated slices on one device; returns (int64 counts[n], probes)."""
    import torch

    S = pb.parallel.routed_slice_nodes(p.n, owners)
    slices = [torch.zeros(S, dtype=torch.int32, device=dev) for _ in range(owners)]
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    for a, b in ranges:
        pb.parallel.count_shard_routed(p, a, b, [t.data_ptr() for t in slices], S, probes=prb, device=dev)
    torch.cuda.synchronize()
    c = torch.cat(slices)
    assert int((c[p.n:] != 0).sum()) == 0  # nothing lands past node n - 1
    return (c[: p.n].to(torch.int64) & 0xFFFFFFFF), int(prb.item())


def _direct_full(p, ranges, dev="cuda:0"):
    import torch

    counts = None
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    for a, b in ranges:
        counts, _ = pb.parallel.count_shard_device(p, p.n, a, b, counts=counts, probes=prb, device=dev)
    torch.cuda.synchronize()
    return (counts.to(torch.int64) & 0xFFFFFFFF), int(prb.item())


@pytest.mark.parametrize("owners", [1, 2, 5])
def test_routed_counts_small_vs_oracle(monkeypatch, owners):
    """The routed count (forced onto the partitioned pass at small n) against
    the oracle: seed graph, ragged ranges, nodes split over 1 / 2 / 5 owners."""
    monkeypatch.setenv("PARBA_FULL_MODE", "partition")
    p = pb.GenParams(n=300_000, d=7, n0=3, seed_edges=TRIANGLE)
    ref = np.zeros(p.n, dtype=np.int64)
    blk, wp = O.generate_block(_op(p), p.m0, p.m)
    O.count_block(ref, blk)
    ranges = [(p.m0, 700_001), (700_001, 700_001), (700_001, p.m)]
    got, pr = _routed_full(p, ranges, owners)
    assert np.array_equal(got.cpu().numpy(), ref) and pr == wp


@pytest.mark.parametrize("env", [{}, {"PARBA_OFF16": "0"}, {"PARBA_ONE_SLICE": "0"}])
def test_routed_counts_large_vs_local(monkeypatch, env):
    """n >= 2^25 (the partitioned pass by default): routed slices over 8
    owners == the local n-word histogram, for the u16-offset, u32-entry and
    multi-slice bucket layouts."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n = 70_000_000 if env.get("PARBA_ONE_SLICE") == "0" else (1 << 25) + 12_345
    p = pb.GenParams(n=n, d=3)
    cut = p.m // 3 + 17
    assert pb.parallel.routed_ok(p, 0, cut) and pb.parallel.routed_ok(p, cut, p.m)
    got, pr = _routed_full(p, [(0, cut), (cut, p.m)], 8)
    monkeypatch.setenv("PARBA_FULL_MODE", "direct")
    want, wp = _direct_full(p, [(0, p.m)])
    assert bool((got == want).all()) and pr == wp
    assert int(got.sum()) == 2 * p.m


def test_routed_counts_validation():
    import torch

    small = pb.GenParams(n=10_000, d=4)
    assert not pb.parallel.routed_ok(small, 0, small.m)
    p = pb.GenParams(n=(1 << 25) + 5, d=2)
    assert pb.parallel.routed_ok(p, 0, p.m) and not pb.parallel.routed_ok(p, 0, 1000)
    S = pb.parallel.routed_slice_nodes(p.n, 2)
    t = [torch.zeros(S, dtype=torch.int32, device="cuda:0") for _ in range(2)]
    ptrs = [x.data_ptr() for x in t]
    with pytest.raises(pb.ParameterError):  # slices too small for n
        pb.parallel.count_shard_routed(p, 0, p.m, ptrs[:1], S)
    with pytest.raises(pb.ParameterError):  # not a multiple of 2^16
        pb.parallel.count_shard_routed(p, 0, p.m, ptrs, S + 1)
    with pytest.raises(pb.ParameterError):  # a shard the partitioned pass does not take
        pb.parallel.count_shard_routed(p, 0, 1000, ptrs, S)
    with pytest.raises(pb.ParameterError):
        pb.parallel.count_shard_routed(p, 0, p.m, [ptrs[0], 0], S)
    pb.parallel.count_shard_routed(p, 5, 5, ptrs, S)  # empty range: nothing to do
    assert int(t[0].sum()) == 0


def test_multi_run_routed_path(monkeypatch):
    """parba_multi_run_shards' owner-routed full histogram, forced on one
    device with three owner slices: equal to the oracle and to the reduce."""
    monkeypatch.setenv("PARBA_FULL_MODE", "partition")
    monkeypatch.setenv("PARBA_MULTI_ROUTED", "1")
    monkeypatch.setenv("PARBA_MULTI_OWNERS", "3")
    p = pb.GenParams(n=200_000, d=6, n0=3, seed_edges=TRIANGLE)
    ref = np.zeros(p.n, dtype=np.int64)
    blk, wp = O.generate_block(_op(p), p.m0, p.m)
    O.count_block(ref, blk)
    got, pr, secs = pb.parallel.multi_run(p, [0, 0, 0], mode="full")
    assert np.array_equal(got, ref) and pr == wp and secs > 0
    monkeypatch.setenv("PARBA_MULTI_ROUTED", "0")
    got2, pr2, _ = pb.parallel.multi_run(p, [0, 0, 0], mode="full")
    assert np.array_equal(got2, ref) and pr2 == wp


def test_multi_run_two_devices():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    p = pb.GenParams(n=10**6, d=8)
    ref, _ = pb.degree_counts(p, workers=1)
    got, st = pb.degree_counts(p, workers=2)
    assert np.array_equal(got.counts, ref.counts) and len(st.per_worker) == 2
    a, _ = pb.run(p, pb.CollectConsumer(), workers=1)
    b, _ = pb.run(p, pb.CollectConsumer(), workers=2)
    assert np.array_equal(a, b)


# --------------------------------------------------------------------------- host-array pipeline


@pytest.mark.parametrize("n,d,n0,lo_frac", [(10**5, 4, 0, 0.0), (3 * 10**6, 11, 3, 0.3), (10**8, 10, 0, 0.9),
                                            (8 * 10**8, 10, 3, 0.9)])
def test_generate_block_host_pipeline(n, d, n0, lo_frac, monkeypatch):
    """Targets-only pipeline == 16-byte-row path == the oracle (several
    chunks, unaligned range starts, seeds)."""
    p = pb.GenParams(n=n, d=d, n0=n0, seed_edges=TRIANGLE if n0 else None)
    lo = p.m0 + int(lo_frac * (p.m - p.m0)) + 3
    hi = min(p.m, lo + 60_000_000)
    got, pr = pb.generate_block(lo, hi, p)
    monkeypatch.setenv("PARBA_HOST_PAIRS", "1")
    rows, pr2 = pb.generate_block(lo, hi, p)
    assert np.array_equal(got, rows) and pr == pr2
    k = min(hi - lo, 2_000_000)
    want, wp = O.generate_block(_op(p), hi - k, hi)
    assert np.array_equal(got[-k:], want)
    ids = np.random.default_rng(3).integers(lo, hi, 4096).astype(np.uint64)
    e, _ = pb.edges_at(ids, p)
    assert np.array_equal(got[ids - np.uint64(lo)], e)


def test_generate_targets_entry_point():
    """parba_generate_targets == the target column of parba_generate; the
    host entry fills unaligned (non-16-byte) host arrays too."""
    import torch

    L = pb._lib.load()
    p = pb.GenParams(n=2 * 10**6, d=9, n0=3, seed_edges=TRIANGLE)
    lo, hi = 12345, p.m - 777
    dev = torch.device("cuda", 0)
    pairs, _ = pb.generate_block_device(lo, hi, p, device=dev)
    t = torch.empty(hi - lo, dtype=torch.int32, device=dev)
    prb = torch.zeros(1, dtype=torch.int64, device=dev)
    pb._lib.check(L.parba_generate_targets(p._device_params(dev), lo, hi, t.data_ptr(), prb.data_ptr(),
                                           pb._lib.stream_ptr(torch, dev)))
    assert torch.equal(t.to(torch.int64) & 0xFFFFFFFF, pairs[:, 1])
    cp, _keep = p._host_params()
    raw = np.zeros(2 * (hi - lo) + 1, dtype=np.uint64)
    out = raw[1:]  # 8-byte aligned only: regular stores
    probes = ctypes.c_uint64(0)
    pb._lib.check(L.parba_generate_host(ctypes.byref(cp), lo, hi, out.ctypes.data, ctypes.byref(probes), 0))
    assert np.array_equal(out.reshape(-1, 2), pairs.cpu().numpy().view(np.uint64))
    s = pb.GenParams(n=1000, d=3, hash=pb.HashConfig(kind=pb.HashKind.SIMPLE))
    with pytest.raises(pb.ParameterError, match="targets-only"):
        pb._lib.check(L.parba_generate_targets(s._device_params(dev), 0, 10, t.data_ptr(), None,
                                               pb._lib.stream_ptr(torch, dev)))


def test_run_workers_with_option_flags_collect_and_file(tmp_path):
    """Node-granular plans (option flags) split over workers: Collect and the
    positional file equal the single-worker result; bb_generate refuses flags."""
    p = pb.GenParams(n=20_000, d=4, n0=10, seed_edges=ring_edges(10), no_self_loops=True, no_parallel_edges=True)
    one, s1 = pb.run(p, pb.CollectConsumer(), workers=1, batch_size=5001)
    three, s3 = pb.run(p, pb.CollectConsumer(), workers=3, batch_size=5001)
    assert np.array_equal(one, three) and s1.hash_probes == s3.hash_probes
    plan = pb.plan_batches(p, 5001)
    assert all((b.lo - p.m0) % 4 == 0 for b in plan)  # node-aligned batches, so node-aligned groups
    path = str(tmp_path / "f.bin")
    with pb.EdgeFileWriter(path, p.m0, p.m - p.m0) as w:
        pb.run(p, w, workers=2, batch_size=3000)
    assert np.array_equal(np.fromfile(path, dtype="<u8").reshape(-1, 2), one)
    with pytest.raises(pb.ParameterError, match="plain mode"):
        pb.bb_generate(p)


def test_multi_run_shards_flags_node_cuts():
    """parba_multi_run_shards with option flags: explicit node-aligned shards
    on one device (repeated) equal the single-range generation and counts."""
    p = pb.GenParams(n=30_000, d=5, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    want, wp = pb.generate_block(p.m0, p.m, p)
    cuts = [p.m0, p.first_edge_of(10_000), p.first_edge_of(20_001), p.m]
    ranges = list(zip(cuts, cuts[1:]))
    rows, prs = pb.parallel.run_shards(p, "store", 0, ranges, [0, 0, 0])
    assert np.array_equal(rows, want) and sum(prs) == wp
    counts, _ = pb.parallel.run_shards(p, "window", 777, ranges, [0, 0, 0])
    ref = np.zeros(777, dtype=np.int64)
    O.count_block(ref, want)
    assert np.array_equal(counts, ref)
