"""GPU parity: the CUDA path (through the C ABI, via the drop-in package)
against the CPU oracle and the golden fixtures made by the reference.

Bar: bit-exact edges, terminal chain values, probe totals and counts.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

import oracle as O
from paper_1602_07106_b200.hashing import HashConfig, HashKind
from conftest import GOLDEN_CRC_N10_D2, GOLDEN_SIMPLE_N10_D2, RING10, TRIANGLE
from powerlaw import attachment_ratios, mle_exponent

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_1602_07106_b200")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _hc(c):
    kind, s0, s1, salt, mult = c
    return pb.HashConfig(kind=pb.HashKind(kind), seed0=s0, seed1=s1, attempt_salt=salt, multiplier=mult)


def _op(p: "pb.GenParams") -> O.OParams:
    s0, s1 = p.hash.crc_seeds()
    return O.OParams(n=p.n, d=p.d, n0=p.n0, seed_edges=tuple(int(x) for x in p.seed_edges),
                     kind=O.KIND_CRC if p.hash.kind is pb.HashKind.CRC else O.KIND_SIMPLE,
                     seed0=p.hash.seed0, seed1=p.hash.seed1, salt=p.hash.attempt_salt,
                     multiplier=p.hash.multiplier)


SEEDS = {"none": (None, 0), "triangle": (TRIANGLE, 3), "ring10": (RING10, 10)}


# --------------------------------------------------------------------------- hashes / chains

def test_hash_all_families_vs_reference_fixture(golden):
    arrays, meta = golden
    rs = arrays["hash_r"]
    for k, c in enumerate(meta["cfgs"]):
        got = pb.hash_many(rs, _hc(c))
        assert np.array_equal(got, arrays[f"hash_out_{k}"]), c


def test_hash_frozen_values_and_edges():
    crc, simple = pb.HashConfig(), pb.HashConfig(kind=pb.HashKind.SIMPLE)
    assert pb.h_crc(3, crc) == 2 and pb.h_crc(1000, crc) == 10 and pb.h_crc(10**6, crc) == 592013
    assert pb.h_crc(1000, pb.HashConfig(seed0=7, seed1=9)) == 96
    assert pb.h_simple(3, simple) == 1 and pb.h_simple(2**32, simple) == 2721204694
    assert pb.h_crc(1, crc) == 0 and pb.h_simple(1, simple) == 0
    with pytest.raises(pb.ParameterError):
        pb.h_crc(0, crc)
    with pytest.raises(pb.ParameterError):
        pb.hash_value(0, simple)


def test_hash_dense_small_r_vs_oracle():
    # every r in [1, 70000) through hash_many (the generic hash kernel:
    # byte-table CRC + mod_int).  The tile kernels' FP64 remainders (mod_fp31,
    # mod_fp, the per-tile reciprocal series) are pinned directly in
    # tests/test_gpu_remainder.py.
    rs = np.arange(1, 70000, dtype=np.uint64)
    for cfg in (pb.HashConfig(), pb.HashConfig(seed0=7, seed1=9, attempt_salt=11)):
        p = O.OParams(n=1, d=1, seed0=cfg.seed0, seed1=cfg.seed1, salt=cfg.attempt_salt)
        assert np.array_equal(pb.hash_many(rs, cfg), O.hash_many(p, rs))


def test_hash_random_wide_r_vs_oracle():
    rng = np.random.default_rng(7)
    for bits in (20, 32, 33, 41, 52, 53, 58, 63, 64):
        rs = rng.integers(1, 2**bits - 1, size=20000, dtype=np.uint64, endpoint=True)
        rs[:3] = [2**bits - 1, 2**(bits - 1), 2**(bits - 1) + 1]
        p = O.OParams(n=1, d=1)
        assert np.array_equal(pb.hash_many(rs, pb.HashConfig()), O.hash_many(p, rs)), bits


def test_chains_vs_reference_fixture(golden):
    arrays, meta = golden
    r0 = arrays["chain_r0"]
    for k, c in enumerate(meta["cfgs"]):
        for stop in (0, 6, 1000):
            vals, probes = pb.resolve_chain_block(r0, stop, _hc(c))
            assert np.array_equal(vals, arrays[f"chain_out_{k}_{stop}"]), (c, stop)
            assert probes == meta["chain_probes"][f"{k}_{stop}"]


def test_resolve_chain_scalar_semantics():
    crc, simple = pb.HashConfig(), pb.HashConfig(kind=pb.HashKind.SIMPLE)
    assert pb.resolve_chain(1, 0, crc) == (0, None, 1)
    assert pb.resolve_chain(11, 0, simple) == (4, None, 2)
    assert pb.resolve_chain(1001, 0, crc) == (286, None, 1)
    cr = pb.resolve_chain(100, 0, crc)  # even start is hashed (body runs at least once)
    assert cr.probes >= 1 and cr.half_pos % 2 == 0
    with pytest.raises(pb.ParameterError):
        pb.resolve_chain(0, 0, crc)
    rng = np.random.default_rng(21)
    saw_seed = False
    for r0 in rng.integers(8, 10_000, size=200):
        cr = pb.resolve_chain(int(r0), 8, crc)
        assert (cr.half_pos is None) != (cr.seed_pos is None)
        saw_seed |= cr.seed_pos is not None
    assert saw_seed


def test_resolve_chain_block_does_not_mutate_and_empty():
    r0 = np.array([5, 7, 9], dtype=np.uint64)
    keep = r0.copy()
    pb.resolve_chain_block(r0, 0, pb.HashConfig())
    assert np.array_equal(r0, keep)
    v, pr = pb.resolve_chain_block(np.empty(0, dtype=np.uint64), 0, pb.HashConfig())
    assert v.size == 0 and pr == 0
    with pytest.raises(pb.ParameterError):
        pb.resolve_chain_block(np.array([0, 3], dtype=np.uint64), 0, pb.HashConfig())


# --------------------------------------------------------------------------- store mode

def test_golden_n10_d2():
    for kind, want in ((pb.HashKind.SIMPLE, GOLDEN_SIMPLE_N10_D2), (pb.HashKind.CRC, GOLDEN_CRC_N10_D2)):
        p = pb.GenParams(n=10, d=2, hash=pb.HashConfig(kind=kind))
        blk, _ = pb.generate_block(0, p.m, p)
        assert [tuple(map(int, r)) for r in blk] == want
        assert [tuple(pb.generate_edge(i, p)) for i in range(20)] == want
        assert [tuple(map(int, r)) for r in pb.edge_list(pb.bb_generate(p))] == want
    assert pb.generate_edge(7, pb.GenParams(n=10, d=2, hash=pb.HashConfig(kind=pb.HashKind.SIMPLE))) == (3, 2)


def test_bb_generate_array_fill(golden):
    """bb_generate: the edge array built by one hash per edge + pointer
    jumping (no chains) equals the chain recomputation of generate_block, the
    oracle's sequential fill and the reference's config-1 sha256, for
    every hash family / seed graph / degree sequence tried."""
    _, meta = golden
    rng = np.random.default_rng(5)
    deg = rng.integers(0, 7, size=50_000).astype(np.uint64)
    fams = [pb.GenParams(n=300_000, d=5), pb.GenParams(n=200_000, d=3, n0=3, seed_edges=TRIANGLE),
            pb.GenParams(n=100_000, d=7, n0=10, seed_edges=RING10,
                         hash=pb.HashConfig(kind=pb.HashKind.SIMPLE)),
            pb.GenParams(n=100_000, d=4, hash=pb.HashConfig(seed0=77, seed1=(1 << 40) + 5, attempt_salt=3)),
            pb.GenParams(n=50_010, n0=10, seed_edges=RING10, degrees=deg)]
    for p in fams:
        e = pb.bb_generate(p)
        assert e.dtype == np.uint64 and e.size == 2 * p.m
        assert np.array_equal(e[: 2 * p.m0], p.seed_edges)
        blk, _ = pb.generate_block(p.m0, p.m, p)
        assert np.array_equal(pb.edge_list(e, p.m0), blk)
        if p.d is not None:
            assert np.array_equal(e, O.bb_generate(_op(p)))
    g = meta["config1"]
    e = pb.bb_generate(pb.GenParams(n=g["n"], d=g["d"]), engine="python")
    assert _sha(e.reshape(-1, 2)) == g["sha256"]
    with pytest.raises(pb.ParameterError, match="uniform degrees only"):
        pb.bb_generate(fams[-1], engine="compiled")
    with pytest.raises(pb.ParameterError, match="rng"):
        pb.bb_generate(fams[0], mode="rng")
    with pytest.raises(pb.ParameterError, match="cap"):
        pb.bb_generate(fams[0], cap=1000)


def test_72_combos_byte_identical(golden):
    _, meta = golden
    for c in meta["combos"]:
        seed, n0 = SEEDS[c["seed"]]
        p = pb.GenParams(n=c["n"], d=c["d"], n0=n0, seed_edges=seed,
                         hash=pb.HashConfig(kind=pb.HashKind(c["kind"])))
        got, probes = pb.generate_block(p.m0, p.m, p)
        assert got.dtype == np.uint64 and got.shape == (p.m - p.m0, 2)
        assert _sha(got) == c["sha256"], c
        assert probes == c["probes"], c


def test_config1_full_array(golden):
    _, meta = golden
    g = meta["config1"]
    p = pb.GenParams(n=g["n"], d=g["d"])
    got, probes = pb.generate_block(0, p.m, p)
    assert _sha(got) == g["sha256"] and probes == g["probes"]
    assert tuple(map(int, got[-1])) == tuple(g["last_edge"])
    want, wp = O.generate_block(_op(p), 0, p.m)
    assert np.array_equal(got, want) and probes == wp
    e = pb.bb_generate(p)
    assert np.array_equal(e.reshape(-1, 2), want)


def test_partition_independence_and_probe_sums():
    rng = np.random.default_rng(24)
    for seed, n0 in ((None, 0), (RING10, 10)):
        p = pb.GenParams(n=30000, d=3, n0=n0, seed_edges=seed)
        whole, probes = pb.generate_block(p.m0, p.m, p)
        cuts = sorted(rng.integers(p.m0, p.m, size=9).tolist())
        bounds = [p.m0] + cuts + [p.m]
        parts = [pb.generate_block(a, b, p) for a, b in zip(bounds, bounds[1:])]
        assert np.array_equal(whole, np.concatenate([x for x, _ in parts]))
        assert probes == sum(pr for _, pr in parts)


def test_unaligned_subranges_vs_oracle():
    rng = np.random.default_rng(5)
    for n, d in ((10**8, 10), (10**9, 100), (10**10, 100), (2**40, 7), (2**55, 4)):
        p = pb.GenParams(n=n, d=d)
        for _ in range(3):
            lo = int(rng.integers(0, p.m - 5000))
            hi = lo + int(rng.integers(1, 5000))
            got, pr = pb.generate_block(lo, hi, p)
            want, wp = O.generate_block(_op(p), lo, hi)
            assert np.array_equal(got, want) and pr == wp, (n, d, lo, hi)
        got, pr = pb.generate_block(p.m - 3000, p.m, p)
        want, wp = O.generate_block(_op(p), p.m - 3000, p.m)
        assert np.array_equal(got, want) and pr == wp


def test_first_probe_series_threshold_vs_oracle():
    """Tiles at and around 2*base = 2^27, where the first probes switch to the
    per-tile reciprocal series, for the 31-bit and the wide remainder paths."""
    for n, d in ((10**8, 10), (10**9, 100), (2**40, 7)):
        p = pb.GenParams(n=n, d=d)
        for c in (1 << 26, 1 << 29):
            lo, hi = c - 4096 - 17, c + 4096 + 5
            assert hi <= p.m
            got, pr = pb.generate_block(lo, hi, p)
            want, wp = O.generate_block(_op(p), lo, hi)
            assert np.array_equal(got, want) and pr == wp, (n, d, c)


def test_sampled_ids_vs_reference_fixture(golden):
    arrays, meta = golden
    for name, s in meta["samples"].items():
        p = pb.GenParams(n=s["n"], d=s["d"])
        ids = arrays[f"sample_{name}_ids"]
        e, probes = pb.edges_at(ids, p)
        assert np.array_equal(e[:, 0], arrays[f"sample_{name}_src"])
        assert np.array_equal(e[:, 1], arrays[f"sample_{name}_tgt"])
        assert probes == int(arrays[f"sample_{name}_probes"].sum())


def test_block_edge_cases():
    p = pb.GenParams(n=10, d=2, n0=3, seed_edges=TRIANGLE)
    arr, pr = pb.generate_block(5, 5, p)
    assert arr.shape == (0, 2) and pr == 0
    for lo, hi in ((0, 5), (5, 18), (9, 5)):
        with pytest.raises(pb.ParameterError):
            pb.generate_block(lo, hi, p)
    with pytest.raises(pb.ParameterError):
        pb.generate_edge(2, p)
    with pytest.raises(pb.ParameterError):
        pb.generate_edge(17, p)
    flagged = pb.GenParams(n=10, d=2, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    with pytest.raises(pb.ParameterError, match="generate_node_edges"):
        pb.generate_edge(3, flagged)
    with pytest.raises(pb.ParameterError, match="node boundary"):
        pb.generate_block(4, 17, flagged)  # flag modes are node-granular
    with pytest.raises(NotImplementedError):  # the base Consumer has no accept (driver.py:70-71)
        pb.run(pb.GenParams(n=10, d=2), pb.Consumer())


def test_node_edges_and_source_law():
    p = pb.GenParams(n=500, d=3, n0=3, seed_edges=TRIANGLE)
    for v in (3, 10, 499):
        first = p.first_edge_of(v)
        assert pb.generate_node_edges(v, p) == [pb.generate_edge(i, p) for i in range(first, first + 3)]
    blk, _ = pb.generate_block(p.m0, p.m, p)
    idx = np.arange(p.m0, p.m, dtype=np.uint64)
    assert np.array_equal(blk[:, 0], (idx - np.uint64(p.m0)) // np.uint64(p.d) + np.uint64(p.n0))
    assert (blk[:, 1] <= blk[:, 0]).all()


def test_store_device_api_and_run_collect():
    import torch

    p = pb.GenParams(n=4000, d=5, n0=3, seed_edges=TRIANGLE)
    want, wp = O.generate_block(_op(p), p.m0, p.m)
    out, probes = pb.generate_block_device(p.m0, p.m, p)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want) and int(probes.item()) == wp
    got, stats = pb.run(p, pb.CollectConsumer(), workers=4, batch_size=64)
    assert np.array_equal(got, want)
    assert stats.edges_emitted == p.m - p.m0 and stats.hash_probes == wp
    n, st = pb.run(p, pb.DiscardConsumer())
    assert n == p.m - p.m0 and st.hash_probes == wp


# --------------------------------------------------------------------------- degree counting

def test_window_subranges_vs_reference_fixture(golden):
    import torch

    arrays, meta = golden
    L = pb._lib.load()
    for w in meta["windows"]:
        p = pb.GenParams(n=w["n"], d=w["d"])
        counts, probes = pb.parallel.count_shard_device(p, w["K"], w["lo"], w["hi"])
        torch.cuda.synchronize()
        c = counts.cpu().numpy()
        assert _sha(c) == w["sha256"], w["name"]
        assert int(probes.item()) == w["probes"]
        assert int(c.sum()) == w["sum"]


def test_degree_counts_vs_reference_fixture(golden):
    arrays, meta = golden
    for f in meta["full"]:
        seed = np.array(f["seed"], dtype=np.uint64) if f["seed"] else None
        p = pb.GenParams(n=f["n"], d=f["d"], n0=f["n0"], seed_edges=seed)
        counter, stats = pb.degree_counts(p)
        assert counter.counts.dtype == np.int64
        assert _sha(counter.counts) == f["sha256"]
        assert int(counter.counts.sum()) == 2 * p.m
        assert stats.hash_probes == f["probes"] and stats.edges_emitted == p.m - p.m0
        # truncated window == prefix of the full count (window kernel vs full kernel)
        win, _ = pb.degree_counts(p, K=777)
        assert np.array_equal(win.counts, counter.counts[:777])


def test_degree_counts_config1(golden):
    _, meta = golden
    g = meta["config1"]
    counter, _ = pb.degree_counts(pb.GenParams(n=g["n"], d=g["d"]))
    assert _sha(counter.counts) == g["counts_sha256"]
    assert counter.counts[:5].tolist() == g["deg0_4"] and int(counter.counts.max()) == g["degree_max"]


def test_full_histogram_n1e6_d16_vs_oracle():
    # config-4 shape at desk scale: exact element-wise counts
    p = pb.GenParams(n=10**6, d=16)
    counter, stats = pb.degree_counts(p)
    blk, wp = O.run_threaded(_op(p), 0, p.m, O.MODE_STORE, threads=os.cpu_count() or 1, batch=1 << 18)
    want = np.bincount(blk.astype(np.int64).ravel(), minlength=p.n)
    assert np.array_equal(counter.counts, want) and stats.hash_probes == wp
    assert 2.6 <= mle_exponent(counter.counts, kmin=16) <= 3.4


def _full_counts(p, lo, hi, mode, monkeypatch):
    import torch

    monkeypatch.setenv("PARBA_FULL_MODE", mode)
    counts, probes = pb.parallel.count_shard_device(p, p.n, lo, hi)
    torch.cuda.synchronize()
    return counts.cpu().numpy(), int(probes.item())


_RAGGED_DEG = np.random.default_rng(7).integers(1, 40, size=200_000)


@pytest.mark.parametrize(
    "case",
    [
        ("n1e6_ragged", dict(n=10**6, d=16), 12345, -777),
        ("tiny_one_bucket", dict(n=1000, d=3), 0, 0),
        ("seeded", dict(n=300_000, d=5, n0=3, seed_edges=TRIANGLE), 3, 0),
        ("all_buckets_one_slice", dict(n=1 << 26, d=2), (1 << 26) - (1 << 22) - 5, 0),
        ("four_slices", dict(n=10**8, d=3), 3 * 10**8 - (1 << 23) - 99, 0),
        ("eight_slices", dict(n=5 * 10**8, d=2), 2 * (5 * 10**8) - (1 << 23) - 99, 0),
        # one-slice buckets (width K / 2048, not a power of two) of the
        # store-targets path: the whole C4 graph, and a seeded ragged range
        ("c4_whole_one_slice", dict(n=10**8, d=16), 0, 0),
        ("one_slice_seeded", dict(n=10**8 + 3, d=2, n0=3, seed_edges=TRIANGLE), 7 * 10**7 + 13, -12345),
        # all-node counts of a graph with 2m >= 2^32 (u64 window, K = n): the
        # wide store-targets pass with FP64 targets, 8 slices per bucket
        ("wide_u64_all_nodes", dict(n=10**9, d=10), (1 << 32) + 5, (1 << 32) + 5 + (1 << 23)),
        # ... and with one scatter pass: the wide store-targets pass (FP64 targets)
        ("wide_u64_store_targets", dict(n=4 * 10**8, d=16), (1 << 32) + 5, (1 << 32) + 5 + (1 << 23)),
        ("simple_hash", dict(n=500_000, d=4, hash=HashConfig(kind=HashKind.SIMPLE, seed0=5)), 0, 0),
        ("degree_sequence", dict(n=3 + _RAGGED_DEG.size, n0=3, degrees=_RAGGED_DEG, seed_edges=TRIANGLE), 3, 0),
    ],
    ids=lambda c: c[0],
)
def test_full_partitioned_equals_direct(case, monkeypatch):
    """The partitioned full histogram (targets -> bucket sort -> shared-memory
    slices, parba_hist.cuh) equals the direct-atomic kernel element-wise,
    probes included, on ragged ranges, seeds, degree sequences, a single
    bucket, every bucket (2048) of one slice, 4 or 8 slices per bucket, and
    the one-slice buckets of the store-targets path (C4)."""
    _, kw, lo, hi = case
    p = pb.GenParams(**kw)
    hi = p.m + hi if hi <= 0 else hi
    part, pp = _full_counts(p, lo, hi, "partition", monkeypatch)
    direct, pd = _full_counts(p, lo, hi, "direct", monkeypatch)
    assert pp == pd
    assert np.array_equal(part, direct)
    assert int(part.astype(np.int64).sum()) == 2 * (hi - lo)
    if case[0] in ("four_slices", "c4_whole_one_slice"):
        # the per-step targets sink (one-slice buckets, u16 offsets), then
        # with 2^k buckets, then with u32 entries in the sorted array
        for env in (("PARBA_STT", "0"), ("PARBA_ONE_SLICE", "0"), ("PARBA_OFF16", "0")):
            monkeypatch.setenv(*env)
            legacy, pl = _full_counts(p, lo, hi, "partition", monkeypatch)
            assert pl == pd and np.array_equal(legacy, direct), env


def test_full_partitioned_vs_oracle_small(monkeypatch):
    # forced partition at desk scale, element-wise against the oracle
    p = pb.GenParams(n=20_000, d=7)
    got, probes = _full_counts(p, 0, p.m, "partition", monkeypatch)
    blk, wp = O.generate_block(_op(p), 0, p.m)
    want = np.bincount(blk.astype(np.int64).ravel(), minlength=p.n)
    assert np.array_equal(got.astype(np.int64), want) and probes == wp


def test_full_partitioned_random_ranges(monkeypatch):
    """Forced partition on 24 seeded random (n, d, seed graph, hash, [lo, hi))
    draws, element-wise against the direct kernel (probes included)."""
    rng = np.random.default_rng(1602)
    for _ in range(24):
        n = int(rng.integers(50, 3_000_000))
        d = int(rng.integers(1, 12))
        kw = dict(n=n, d=d)
        if rng.random() < 0.3:
            kw.update(n0=3, seed_edges=TRIANGLE)
        if rng.random() < 0.3:
            kw.update(hash=HashConfig(kind=HashKind.SIMPLE, seed0=int(rng.integers(0, 1 << 32))))
        p = pb.GenParams(**kw)
        lo = int(rng.integers(p.m0, p.m))
        hi = int(rng.integers(lo, p.m + 1))
        part, pp = _full_counts(p, lo, hi, "partition", monkeypatch)
        direct, pd = _full_counts(p, lo, hi, "direct", monkeypatch)
        assert pp == pd and np.array_equal(part, direct), (kw, lo, hi)


def test_partitioned_counts_accumulate(monkeypatch):
    """parba_degree_full / parba_degree_window add into the caller's counts
    (+=, the reference's Consumer.merge) on the partitioned path too."""
    import torch

    monkeypatch.setenv("PARBA_FULL_MODE", "partition")
    p = pb.GenParams(n=300_000, d=9)
    lo, hi = 1000, p.m - 1000
    once, _ = pb.parallel.count_shard_device(p, p.n, lo, hi)
    pre = torch.arange(p.n, dtype=torch.int32, device="cuda") % 7
    acc, _ = pb.parallel.count_shard_device(p, p.n, lo, hi, counts=pre.clone())
    assert torch.equal(acc, once + pre)
    K = 200_000
    w_once, _ = _window_counts(p, K, lo, hi, "partition", monkeypatch)
    base = torch.arange(K, dtype=torch.int64, device="cuda")
    probes = torch.zeros(1, dtype=torch.int64, device="cuda")
    w_acc, _ = pb.parallel.count_shard_device(p, K, lo, hi, counts=base.clone(), probes=probes)
    assert torch.equal(w_acc, w_once + base)


def test_full_partitioned_multi_pass(monkeypatch):
    # n > 2048 * 2^18: 2289 buckets of 8 slices, scattered in two passes
    p = pb.GenParams(n=6 * 10**8, d=2)
    lo = p.m - (1 << 22)
    part, pp = _full_counts(p, lo, p.m, "partition", monkeypatch)
    direct, pd = _full_counts(p, lo, p.m, "direct", monkeypatch)
    assert pp == pd and np.array_equal(part, direct)


def _window_counts(p, K, lo, hi, mode, monkeypatch):
    import torch

    monkeypatch.setenv("PARBA_FULL_MODE", mode)
    counts = torch.zeros(K, dtype=torch.int64, device="cuda")
    probes = torch.zeros(1, dtype=torch.int64, device="cuda")
    pb.parallel.count_shard_device(p, K, lo, hi, counts=counts, probes=probes)
    torch.cuda.synchronize()
    return counts, int(probes.item())


@pytest.mark.parametrize(
    "case",
    [
        ("half_window", dict(n=10**6, d=8), 500_000, 777, -3),
        ("one_node", dict(n=10**6, d=8), 1, 0, 0),
        ("slice_plus_one", dict(n=10**6, d=3), (1 << 15) + 1, 5, -5),
        ("seeded_degseq", dict(n=3 + _RAGGED_DEG.size, n0=3, degrees=_RAGGED_DEG, seed_edges=TRIANGLE), 150_000, 3, 0),
        ("two_passes_u64", dict(n=10**9, d=10), 10**9, -(1 << 23), 0),
        ("max_domain_2p31", dict(n=2**31 + 5, d=2), 2**31, -(1 << 22), 0),
        ("beyond_domain_direct", dict(n=2**31 + 5, d=2), 2**31 + 1, -(1 << 22), 0),
        ("n_above_2p32", dict(n=6 * 10**9, d=2), 10**8, -(1 << 22), 0),
    ],
    ids=lambda c: c[0],
)
def test_window_partitioned_equals_direct(case, monkeypatch):
    """u64 degree windows through the partitioned pass (targets < K kept;
    several scatter passes above 2048 buckets) equal the window kernel."""
    import torch

    _, kw, K, lo, hi = case
    p = pb.GenParams(**kw)
    lo = p.m + lo if lo < 0 else lo
    hi = p.m + hi if hi <= 0 else hi
    part, pp = _window_counts(p, K, lo, hi, "partition", monkeypatch)
    direct, pd = _window_counts(p, K, lo, hi, "direct", monkeypatch)
    assert pp == pd and torch.equal(part, direct)
    del part, direct


def test_window_large_range_sharding_independent():
    # C3 shape: n=1e9, d=100, K=1e5 over the first 1e9 edge IDs; any split of
    # the range into shards sums to the same histogram
    import torch

    p = pb.GenParams(n=10**9, d=100)
    lo, hi, K = 0, 10**9, 10**5
    whole, pr = pb.parallel.count_shard_device(p, K, lo, hi)
    for G in (2, 3, 8):
        acc = torch.zeros_like(whole)
        prs = torch.zeros_like(pr)
        for g in range(G):
            a, b = pb.parallel.shard_range(lo, hi, g, G)
            pb.parallel.count_shard_device(p, K, a, b, counts=acc, probes=prs)
        torch.cuda.synchronize()
        assert torch.equal(acc, whole) and int(prs.item()) == int(pr.item())
    # sources of edges < K*d = 1e7 all land in the window: K*d each
    c = whole.cpu().numpy()
    assert (c >= 100).all()  # every node < K owns its d = 100 edges in [0, 1e9)
    assert 1.9 <= int(pr.item()) / (hi - lo) <= 2.1


@pytest.mark.parametrize("cfg", [("C3", 10**9, 100), ("C5", 10**10, 100)], ids=lambda c: c[0])
def test_full_baseline_window_independent_of_gpu_count(cfg):
    """The whole C3 (1e11 edges) and C5 (1e12 edges) windows (K = 1e5): the
    8-way edge-ID partition's per-shard counts sum to the single-range run,
    probes included (identical for G in {1, 2, 4, 8}), and the
    window holds every source of its K*d edges."""
    import torch

    _, n, d = cfg
    p = pb.GenParams(n=n, d=d)
    K = 10**5
    whole, pr = pb.parallel.count_shard_device(p, K, 0, p.m)
    acc = torch.zeros_like(whole)
    prs = torch.zeros_like(pr)
    for g in range(8):
        a, b = pb.parallel.shard_range(0, p.m, g, 8)
        pb.parallel.count_shard_device(p, K, a, b, counts=acc, probes=prs)
    torch.cuda.synchronize()
    assert torch.equal(acc, whole) and int(prs.item()) == int(pr.item())
    c = whole.cpu().numpy()
    assert (c >= d).all() and 1.99 <= int(pr.item()) / p.m <= 2.01


def test_probe_cost_per_edge():
    # acceptance (3): mean probes/edge in [1.8, 2.2]
    for kind in (pb.HashKind.CRC, pb.HashKind.SIMPLE):
        p = pb.GenParams(n=600_000, d=2, hash=pb.HashConfig(kind=kind))
        _, probes = pb.generate_block(10**5, 10**5 + 10**6, p)
        assert 1.8 <= probes / 10**6 <= 2.2


def test_expected_degree_law_billion_edges():
    # acceptance (6): n=1e7, d=100, K=1e4, SIMPLE, 1e9 edges
    n, d, K = 10**7, 100, 10**4
    p = pb.GenParams(n=n, d=d, hash=pb.HashConfig(kind=pb.HashKind.SIMPLE))
    counter, stats = pb.degree_counts(p, K=K)
    ratios = attachment_ratios(counter.counts, n=n, d=d, bins=12, lo=10, hi=K)
    assert len(ratios) >= 10 and all(0.8 <= r <= 1.2 for r in ratios)
    assert stats.edges_emitted == 10**9


def test_degree_conservation_randomized():
    rng = np.random.default_rng(90)
    for case in range(20):
        n0 = int(rng.integers(0, 6))
        seed = None
        if n0 >= 2:
            flat = list(RING10[:0])
            for i in range(n0):
                flat += (i, (i + 1) % n0)
            for _ in range(int(rng.integers(0, 5))):
                flat += (int(rng.integers(n0)), int(rng.integers(n0)))
            seed = np.array(flat, dtype=np.uint64)
        else:
            n0 = 0
        kind = pb.HashKind.CRC if rng.random() < 0.5 else pb.HashKind.SIMPLE
        p = pb.GenParams(n=int(rng.integers(n0 + 1, 4000)), d=int(rng.integers(1, 9)), n0=n0,
                         seed_edges=seed, hash=pb.HashConfig(kind=kind))
        counter, _ = pb.degree_counts(p)
        assert int(counter.counts.sum()) == 2 * p.m
        want = np.zeros(p.n, dtype=np.int64)
        blk, _ = O.generate_block(_op(p), p.m0, p.m)
        O.count_block(want, blk)
        if p.m0:
            O.count_block(want, p.seed_edges.reshape(-1, 2))
        assert np.array_equal(counter.counts, want)


# --------------------------------------------------------------------------- full BASELINE sizes

def test_config2_full_size_properties():
    """C2 (n=1e8, d=10, m=1e9; 16 GB in HBM): closed-form sources over the
    whole array, target <= source, 1e6 sampled rows bit-exact vs the oracle,
    probe mean, and the device histogram of the stored targets equals the
    fused full-count kernel (a checksum of two independent kernels)."""
    import torch

    p = pb.GenParams(n=10**8, d=10)
    out, probes = pb.generate_block_device(0, p.m, p)
    torch.cuda.synchronize()
    step = 1 << 27
    for a in range(0, p.m, step):
        b = min(a + step, p.m)
        src = out[a:b, 0]
        idx = torch.arange(a, b, dtype=torch.int64, device=out.device)
        assert torch.equal(src, idx // p.d)
        assert bool((out[a:b, 1] <= src).all())
    rng = np.random.default_rng(160207106)
    ids = np.unique(rng.integers(0, p.m, size=10**6, dtype=np.uint64))  # 1e6 sampled IDs
    rows = out[torch.from_numpy(ids.view(np.int64)).to(out.device)].cpu().numpy().view(np.uint64)
    r0 = np.uint64(2) * ids + np.uint64(1)
    term, _ = O.resolve_chain_block(_op(p), r0, 0)
    assert np.array_equal(rows[:, 0], ids // np.uint64(10))
    assert np.array_equal(rows[:, 1], (term >> np.uint64(1)) // np.uint64(10))
    assert 1.95 <= int(probes.item()) / p.m <= 2.05
    tgt_hist = torch.bincount(out[:, 1], minlength=p.n)
    del out
    counts, pr2 = pb.parallel.count_shard_device(p, p.n, 0, p.m)
    torch.cuda.synchronize()
    c64 = pb.parallel.widen_counts(torch, counts, p.n)
    assert int(pr2.item()) == int(probes.item())
    assert torch.equal(c64 - p.d, tgt_hist)  # every node is the source of exactly d edges
    assert int(c64.sum().item()) == 2 * p.m


def test_config4_full_histogram_properties():
    """C4 (n=1e8, d=16, m=1.6e9, uint32 counts): sum = 2m, min degree d,
    power-law exponent in range, and the counts of a node subrange equal the
    window kernel's."""
    import torch

    p = pb.GenParams(n=10**8, d=16)
    counts, probes = pb.parallel.count_shard_device(p, p.n, 0, p.m)
    c64 = pb.parallel.widen_counts(torch, counts, p.n)
    assert int(c64.sum().item()) == 2 * p.m
    assert int(c64.min().item()) >= p.d
    win, _ = pb.parallel.count_shard_device(p, 100_000, 0, p.m)
    torch.cuda.synchronize()
    assert torch.equal(win[:100_000], c64[:100_000])
    assert 2.6 <= mle_exponent(c64.cpu().numpy(), kmin=32) <= 3.4


# --------------------------------------------------------------------------- binary file writer (f2)

def test_binary_file_equals_oracle_and_is_schedule_independent(tmp_path):
    import hashlib as _h

    from paper_1602_07106_b200 import io as pio

    p = pb.GenParams(n=10**5, d=8)  # reference acceptance (2): n=1e5, d=8
    want, _ = O.generate_block(_op(p), 0, p.m)
    path = tmp_path / "edges.bin"
    nbytes, probes = pb.write_edges_binary(str(path), p)
    data = path.read_bytes()
    assert nbytes == len(data) == 16 * p.m
    assert data == np.ascontiguousarray(want, dtype="<u8").tobytes()
    digests = {_h.sha256(data).hexdigest()}
    old = pio.FILE_CHUNK_EDGES
    try:
        for chunk in (1 << 10, 12345):
            pio.FILE_CHUNK_EDGES = chunk
            w = pb.EdgeFileWriter(str(path), p.m0, p.m - p.m0)
            merged, stats = pb.run(p, w, workers=4, batch_size=1 << 10)
            w.close()
            assert merged == 16 * p.m and stats.hash_probes == probes
            digests.add(_h.sha256(path.read_bytes()).hexdigest())
    finally:
        pio.FILE_CHUNK_EDGES = old
    assert len(digests) == 1
    # seeded family, partial range written by two "workers" in reverse order
    q = pb.GenParams(n=3000, d=3, n0=10, seed_edges=RING10)
    w = pb.EdgeFileWriter(str(path), q.m0, q.m - q.m0)
    mid = (q.m0 + q.m) // 2 + 1
    w.write_range(q, mid, q.m)
    w.write_range(q, q.m0, mid)
    w.close()
    blk, _ = O.generate_block(_op(q), q.m0, q.m)
    assert path.read_bytes() == np.ascontiguousarray(blk, dtype="<u8").tobytes()


def test_binary_file_native_writer_vs_pwrite(tmp_path, monkeypatch):
    """parba_write_binary (the file range mapped and filled by the host
    pipeline) writes the same bytes as the pinned-buffer pwrite path, for the
    targets pipeline (CRC) and the 16-byte-row pipeline (SIMPLE hash, option
    flags), at page-misaligned offsets, and refuses ranges outside the file."""
    import ctypes

    from paper_1602_07106_b200 import _lib

    fams = [pb.GenParams(n=3 * 10**6, d=7),
            pb.GenParams(n=2 * 10**5, d=5, hash=HashConfig(kind=HashKind.SIMPLE, seed0=77)),
            pb.GenParams(n=10**5, d=4, n0=3, seed_edges=TRIANGLE, no_self_loops=True)]
    for k, p in enumerate(fams):
        a = p.m0 + 12345 if p.d is not None and not p.no_self_loops else p.m0
        b = p.m - 777 if not p.no_self_loops else p.m
        paths = []
        # mapped range, staged buffers + pwrite (native), pinned buffers + pwrite (Python)
        for mode, mm in (("0", "1"), ("0", "0"), ("1", None)):
            monkeypatch.setenv("PARBA_WRITER_PWRITE", mode)
            if mm is None:
                monkeypatch.delenv("PARBA_WRITER_MMAP", raising=False)
            else:
                monkeypatch.setenv("PARBA_WRITER_MMAP", mm)
            path = tmp_path / f"w{k}_{mode}{mm}.bin"
            with pb.EdgeFileWriter(str(path), p.m0, p.m - p.m0) as w:
                nb, pr = w.write_range(p, a, b)
            assert nb == 16 * (b - a)
            paths.append((path, pr))
        assert len({q.read_bytes() for q, _ in paths}) == 1 and len({pr for _, pr in paths}) == 1
        op = _op(p)
        if p.no_self_loops:
            op = O.OParams(n=p.n, d=p.d, n0=p.n0, seed_edges=tuple(int(x) for x in p.seed_edges),
                           no_self_loops=True)
        want, wp = O.generate_block(op, a, b)
        got = np.fromfile(paths[0][0], dtype="<u8").reshape(-1, 2)[a - p.m0: b - p.m0]
        assert np.array_equal(got, want) and paths[0][1] == wp
    monkeypatch.delenv("PARBA_WRITER_PWRITE")
    monkeypatch.delenv("PARBA_WRITER_MMAP", raising=False)
    p = fams[0]
    # a write-only descriptor cannot be mapped: the staged pwrite path takes over
    import os as _os

    path = tmp_path / "wo.bin"
    fd = _os.open(str(path), _os.O_WRONLY | _os.O_CREAT | _os.O_TRUNC, 0o644)
    _os.ftruncate(fd, 16 * 100_000)
    cp, _keep = p._host_params()
    pr = ctypes.c_uint64(0)
    monkeypatch.setenv("PARBA_WRITER_MMAP", "1")  # the mapped path is asked for and refused
    assert _lib.load().parba_write_binary(ctypes.byref(cp), 0, 100_000, fd, 0, ctypes.byref(pr), 0) == 0
    monkeypatch.delenv("PARBA_WRITER_MMAP")
    _os.close(fd)
    want, wp = O.generate_block(_op(p), 0, 100_000)
    assert np.array_equal(np.fromfile(path, dtype="<u8").reshape(-1, 2), want) and pr.value == wp
    path = tmp_path / "short.bin"
    with pb.EdgeFileWriter(str(path), p.m0, 1000) as w:
        with pytest.raises(pb.ParameterError):
            w.write_range(p, 0, 2000)
        cp, _keep = p._host_params()
        rc = _lib.load().parba_write_binary(ctypes.byref(cp), 0, 2000, w.fd, 0, None, 0)
        assert rc != 0 and b"range needs" in _lib.load().parba_last_error()


# --------------------------------------------------------------------------- C ABI, host-buffer entry points

def test_c_abi_host_entry_points():
    import ctypes

    from paper_1602_07106_b200 import _lib, hashing

    L = _lib.load()
    # seeded family: the _host variants take a HOST seed pointer
    seed = np.ascontiguousarray(RING10, dtype=np.uint64)
    p = pb.GenParams(n=5000, d=4, n0=10, seed_edges=seed)
    cp = hashing.c_params(p.hash, p.n, p.d, p.n0, p.m0, seed.ctypes.data)
    lo, hi = p.m0 + 7, p.m - 3
    out = np.empty((hi - lo, 2), dtype=np.uint64)
    probes = ctypes.c_uint64(0)
    rc = L.parba_generate_host(ctypes.byref(cp), lo, hi, out.ctypes.data, ctypes.addressof(probes), 0)
    assert rc == 0, L.parba_last_error()
    want, wp = O.generate_block(_op(p), lo, hi)
    assert np.array_equal(out, want) and probes.value == wp
    K = 777
    counts = np.full(K, 5, dtype=np.int64)  # accumulates (+=)
    rc = L.parba_degree_window_host(ctypes.byref(cp), p.m0, p.m, K, counts.ctypes.data,
                                    ctypes.addressof(probes), 0)
    assert rc == 0, L.parba_last_error()
    ref = np.zeros(K, dtype=np.int64)
    blk, _ = O.generate_block(_op(p), p.m0, p.m)
    O.count_block(ref, blk)
    assert np.array_equal(counts, ref + 5)
    # errors map to status codes, no exception crosses the ABI
    assert L.parba_generate_host(ctypes.byref(cp), 0, 5, out.ctypes.data, None, 0) == _lib.PARBA_EINVAL
    assert b"out of range" in L.parba_last_error()


def test_multi_run_single_process_shards():
    """parba_multi_run (one process, a host thread per device; here the same
    GPU three times): every mode equals the single-device result."""
    import oracle as O

    p = pb.GenParams(n=20000, d=5, n0=3, seed_edges=TRIANGLE)
    want, wp = pb.generate_block(p.m0, p.m, p)
    got, pr, secs = pb.parallel.multi_run(p, [0, 0, 0], mode="store")
    assert np.array_equal(got, want) and pr == wp and secs > 0
    full, fp = pb.degree_counts(p)
    got, pr, _ = pb.parallel.multi_run(p, [0, 0], mode="full")
    seed_counts = np.bincount(TRIANGLE.astype(np.int64), minlength=p.n)
    assert np.array_equal(got + seed_counts, full.counts) and pr == wp
    got, pr, _ = pb.parallel.multi_run(p, [0, 0, 0], mode="window", K=777)
    assert np.array_equal(got + seed_counts[:777], full.counts[:777])
    _, pr, _ = pb.parallel.multi_run(p, [0, 0], mode="discard")
    assert pr == wp
    f = pb.GenParams(n=5000, d=3, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    fw, fwp = pb.generate_block(f.m0, f.m, f)
    got, pr, _ = pb.parallel.multi_run(f, [0, 0, 0], mode="store")  # node-aligned shards
    assert np.array_equal(got, fw) and pr == fwp
    big = pb.GenParams(n=10**9, d=100)
    with pytest.raises(pb.ParameterError, match="2m < 2"):
        pb.parallel.multi_run(big, [0], mode="full")


def test_crc_primitive_and_vector_helpers(golden):
    """crc32c_u64(_many), mulhi_u64, h_crc_many / h_simple_many (hashing.py:
    105-198) on the device vs the reference's fixture and exact integers."""
    arrays, meta = golden
    seeds, words, want = arrays["crc_seeds"], arrays["crc_words"], arrays["crc_out"]
    got = np.array([pb.crc32c_u64_many(int(s), np.array([w]))[0] for s, w in zip(seeds, words)], dtype=np.uint64)
    assert np.array_equal(got, want)
    assert pb.crc32c_u64(int(seeds[0]), int(words[0])) == int(want[0])
    for s in (0, 1, 0xFFFFFFFF):
        batch = pb.crc32c_u64_many(s, words)
        assert np.array_equal(batch[:4], [O.crc32c_u64(s, int(w)) for w in words[:4]])
    rng = np.random.default_rng(9)
    a = rng.integers(0, 2**64 - 1, size=5000, dtype=np.uint64, endpoint=True)
    b = rng.integers(0, 2**64 - 1, size=5000, dtype=np.uint64, endpoint=True)
    hi = pb.mulhi_u64(a, b)
    assert all(int(h) == (int(x) * int(y)) >> 64 for h, x, y in zip(hi[:500], a[:500], b[:500]))
    rs = arrays["hash_r"]
    for k, c in enumerate(meta["cfgs"]):
        f = pb.h_crc_many if c[0] == "crc" else pb.h_simple_many
        assert np.array_equal(f(rs, _hc(c)), arrays[f"hash_out_{k}"]), c
    from paper_1602_07106_b200 import _kernels

    _kernels.warmup()
    vals, pr = _kernels.resolve_chain_block(np.array([1001], dtype=np.uint64), 0, pb.HashConfig())
    assert pr >= 1 and int(vals[0]) % 2 == 0


# --------------------------------------------------------------------------- generic consumers
# (reference tests/test_driver.py:160-270 restated: user plug-ins run the
# batch loop with host-thread workers; every batch is generated on the GPU)

class _Exploding(pb.Consumer):
    def new_context(self, worker_id):
        return 0

    def accept_block(self, ctx, lo, edges):
        raise RuntimeError("synthetic consumer failure")

    def merge(self, contexts):
        return None


class _PerEdgeSum(pb.Consumer):
    def new_context(self, worker_id):
        return {"sum": 0, "count": 0}

    def accept(self, ctx, i, edge):
        ctx["sum"] += edge.source + edge.target
        ctx["count"] += 1

    def merge(self, contexts):
        return sum(c["sum"] for c in contexts), sum(c["count"] for c in contexts)


class _Bitmap(pb.Consumer):
    def __init__(self, m0, m):
        self.m0, self.m = m0, m

    def new_context(self, worker_id):
        return np.zeros(self.m - self.m0, dtype=np.int64)

    def accept_block(self, ctx, lo, edges):
        ctx[lo - self.m0: lo - self.m0 + edges.shape[0]] += 1
        return ctx

    def merge(self, contexts):
        return sum(contexts)


class _Sleepy(pb.Consumer):
    def __init__(self, slow_lo):
        self.slow_lo = slow_lo

    def new_context(self, worker_id):
        return 0

    def accept_block(self, ctx, lo, edges):
        import time

        if lo == self.slow_lo:
            time.sleep(0.6)
        return ctx + 1

    def merge(self, contexts):
        return list(contexts)


def test_generic_consumers_batch_loop():
    p = pb.GenParams(n=100, d=2)
    arr, _ = pb.run(p, pb.CollectConsumer())
    want = (int(arr.sum()), p.m)
    assert pb.run(p, _PerEdgeSum(), workers=1, batch_size=17)[0] == want
    assert pb.run(p, _PerEdgeSum(), workers=2, batch_size=17)[0] == want
    q = pb.GenParams(n=500, d=3, n0=3, seed_edges=TRIANGLE)
    for workers in (1, 3):
        seen, st = pb.run(q, _Bitmap(q.m0, q.m), workers=workers, batch_size=97)
        assert (seen == 1).all() and st.edges_emitted == q.m - q.m0
        _, wp = O.generate_block(_op(q), q.m0, q.m)
        assert st.hash_probes == wp
    with pytest.raises(pb.GenerationError, match="worker .* failed") as ei:
        pb.run(q, _Exploding(), workers=2, batch_size=10)
    assert "synthetic consumer failure" in str(ei.value)
    with pytest.raises(RuntimeError, match="synthetic consumer failure"):
        pb.run(q, _Exploding(), workers=1)
    r = pb.GenParams(n=40, d=3, n0=3, seed_edges=TRIANGLE)  # 111 edges, 12 batches
    counts, st = pb.run(r, _Sleepy(r.m0), workers=2, batch_size=10)
    assert sum(counts) == 12 and max(counts) >= 10
    assert sum(w.batches for w in st.per_worker) == 12
    # option flags: node-granular batches through a generic consumer
    f = pb.GenParams(n=300, d=3, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    seen, _ = pb.run(f, _Bitmap(f.m0, f.m), workers=2, batch_size=10)
    assert (seen == 1).all()


def test_huge_degree_and_offsets_vs_oracle():
    """Closed forms with d >= 2^31 (the narrow 32-bit division does not
    apply) and large seed offsets, store and window, vs the oracle."""
    seed = np.array([x for i in range(50) for x in (i, (i + 7) % 50)], dtype=np.uint64)
    for n, d, n0, sd in ((4, 2**33 + 7, 0, None), (60, 3 * 2**31, 50, seed), (10**6, 2**31 - 1, 50, seed)):
        p = pb.GenParams(n=n, d=d, n0=n0, seed_edges=sd)
        op = _op(p)
        rng = np.random.default_rng(d % 1000)
        for _ in range(3):
            lo = int(rng.integers(p.m0, p.m - 3000))
            hi = lo + 3000
            got, pr = pb.generate_block(lo, hi, p)
            want, wp = O.generate_block(op, lo, hi)
            assert np.array_equal(got, want) and pr == wp, (n, d, lo)
            K = n0 + 2
            import torch

            c, prb = pb.parallel.count_shard_device(p, K, lo, hi)
            torch.cuda.synchronize()
            w, _ = O.degree_block(op, lo, hi, K)
            assert np.array_equal(c.cpu().numpy()[:K], w), (n, d, lo, "window")


def test_wide_store_flush_with_seed_vs_oracle():
    """Store tiles at positions >= 2^32 (64-bit chain values) with and
    without a seed graph: the per-tile source division path of the flush."""
    seed = np.array([x for i in range(40) for x in (i, (i + 3) % 40)], dtype=np.uint64)
    for n0, sd in ((0, None), (40, seed)):
        p = pb.GenParams(n=10**9, d=10, n0=n0, seed_edges=sd)
        op = _op(p)
        for lo in (5 * 10**9 + 13, 2**33 - 1000):
            hi = lo + 70_000
            got, pr = pb.generate_block(lo, hi, p)
            want, wp = O.generate_block(op, lo, hi)
            assert np.array_equal(got, want) and pr == wp, (n0, lo)


def test_config5_ten_million_sampled_ids_vs_oracle():
    """SURVEY 8d, configs[4] (n=1e10, d=100, m=1e12): 1e7 uniformly sampled
    edge IDs through the device chain kernel vs the oracle's chains."""
    p = pb.GenParams(n=10**10, d=100)
    rng = np.random.default_rng(160207106)
    ids = rng.integers(0, p.m, size=10**7, dtype=np.uint64)
    e, probes = pb.edges_at(ids, p)
    term, wp = O.resolve_chain_block(_op(p), np.uint64(2) * ids + np.uint64(1), 0)
    assert np.array_equal(e[:, 0], ids // np.uint64(100))
    assert np.array_equal(e[:, 1], (term >> np.uint64(1)) // np.uint64(100))
    assert probes == wp


def test_config3_window_subranges_1e8_vs_oracle():
    """SURVEY 8d, configs[2] (n=1e9, d=100, K=1e5): window counts of the
    1e8-edge subranges [0, 1e8) (every source hit) and [m - 1e8, m) vs the
    threaded oracle."""
    import os

    import torch

    p = pb.GenParams(n=10**9, d=100)
    K = 10**5
    threads = max(1, len(os.sched_getaffinity(0)))
    for lo in (0, p.m - 10**8):
        hi = lo + 10**8
        c, prb = pb.parallel.count_shard_device(p, K, lo, hi)
        torch.cuda.synchronize()
        want, wp = O.run_threaded(_op(p), lo, hi, O.MODE_WINDOW, K=K, threads=threads, batch=1 << 20)
        assert np.array_equal(c.cpu().numpy()[:K], want) and int(prb.item()) == wp, lo


@pytest.mark.parametrize("seeded", [False, True])
def test_wide_store_vs_oracle(seeded):
    """Wide store launches (chain values >= 2^32, 64-bit stage and queue
    entries) on ragged ranges, with and without a seed graph, vs the oracle;
    also a range straddling 2^31 positions (two launch widths)."""
    import torch

    if seeded:
        p = pb.GenParams(n=8 * 10**8 + 3, d=10, n0=3, seed_edges=TRIANGLE)
    else:
        p = pb.GenParams(n=8 * 10**8, d=10)
    dev = torch.device("cuda", 0)
    for lo, hi in ((7 * 10**9 + 11, 7 * 10**9 + 3_000_013), (p.m - 2_000_001, p.m),
                   ((1 << 31) - 777, (1 << 31) + 1_000_000)):
        got, prb = pb.generate_block_device(lo, hi, p, device=dev)
        g = got.cpu().numpy().view(np.uint64)
        want, wp = O.generate_block(_op(p), lo, hi)
        assert np.array_equal(g, want) and int(prb.item()) == wp


@pytest.mark.parametrize("n,d,seeded", [((1 << 32), 174761, False), ((1 << 32) - 1, 3, True),
                                        (10**9, 174761, True), (3 * 10**9, 1000, False), (10**9, 174762, False)])
def test_wide_store_fp64_targets_at_the_bounds(n, d, seeded, monkeypatch):
    """Wide store targets by the FP64 reciprocal (target_fp: n <= 2^32,
    d < 174762) at the edges of its range, and d = 174762 (integer path),
    vs the oracle and vs the 64-bit integer division (PARBA_TGT_FP=0)."""
    import torch

    kw = dict(n0=3, seed_edges=TRIANGLE) if seeded else {}
    p = pb.GenParams(n=n, d=d, **kw)
    dev = torch.device("cuda", 0)
    for lo, hi in ((p.m - 600_017, p.m), (p.m // 2 - 300_000, p.m // 2 + 300_001)):
        got, prb = pb.generate_block_device(lo, hi, p, device=dev)
        g = got.cpu().numpy().view(np.uint64)
        want, wp = O.generate_block(_op(p), lo, hi)
        assert np.array_equal(g, want) and int(prb.item()) == wp, (lo, hi)
        monkeypatch.setenv("PARBA_TGT_FP", "0")
        alt, _ = pb.generate_block_device(lo, hi, p, device=dev)
        monkeypatch.delenv("PARBA_TGT_FP")
        assert np.array_equal(alt.cpu().numpy().view(np.uint64), g)


@pytest.mark.parametrize("hi", [1 << 30, (1 << 30) + 1, (1 << 30) + 100, 0x78000000, 0x78000000 + 1, 1 << 31,
                                (1 << 31) + 1, (1 << 31) + 77])
def test_chunk_class_boundaries(hi):
    """The launch's kernel class follows its largest chain value 2*hi-1:
    ranges ending at exactly 2^30 / 0x78000000 edges run the 2- / 3-chunk
    kernels (r < 2^31 / r <= 0xF0000000, the 32-bit-tail remainder's range),
    one edge more the next class.  Store, window and
    full counts of [hi - 300017, hi) vs the oracle, ragged top tiles included."""
    import torch

    p = pb.GenParams(n=27 * 10**7, d=8)
    op = _op(p)
    dev = torch.device("cuda", 0)
    lo = hi - 300_017
    got, prb = pb.generate_block_device(lo, hi, p, device=dev)
    want, wp = O.generate_block(op, lo, hi)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want) and int(prb.item()) == wp
    K = 10**5
    counts, cprb = pb.parallel.count_shard_device(p, K, lo, hi, device=dev)
    w, _ = O.degree_block(op, lo, hi, K)
    assert np.array_equal(counts.cpu().numpy(), w) and int(cprb.item()) == wp
    # all nodes (2m >= 2^32 here: the u64 window kernel with K = n)
    full, _ = pb.parallel.count_shard_device(p, p.n, lo, hi, device=dev)
    nodes, cnt = np.unique(want.reshape(-1), return_counts=True)
    idx = torch.from_numpy(nodes.astype(np.int64)).to(dev)
    assert np.array_equal(full[idx].cpu().numpy(), cnt) and int(full.sum().item()) == 2 * (hi - lo)
