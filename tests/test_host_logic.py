"""Host-side logic of the drop-in package (CPU only): configuration objects,
validation and error behaviour mirror the reference (hashing.py:48-85,
generator.py:50-136, driver.py:131-158)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1602_07106_b200 as pb
from conftest import TRIANGLE, ring_edges


def test_hash_config_validation_and_folding():
    for kw in ({"seed0": -1}, {"seed1": 2**64}, {"kind": pb.HashKind.SIMPLE, "multiplier": 2**64}):
        with pytest.raises(pb.ParameterError):
            pb.HashConfig(**kw)
    with pytest.raises(pb.ParameterError):
        pb.HashConfig().with_attempt(-1)
    cfg = pb.HashConfig(seed0=10, seed1=20)
    assert cfg.crc_seeds() == (10, 20)
    assert cfg.with_attempt(3).crc_seeds() == (13, (20 + 3 * 0x9E3779B9) & 0xFFFFFFFF)
    assert pb.HashConfig(seed0=2**40 + 5).crc_seeds()[0] == 5  # seeds are 32-bit
    mults = {pb.HashConfig(kind=pb.HashKind.SIMPLE).with_attempt(a).simple_multiplier() for a in range(12)}
    assert len(mults) == 12 and all(m & 1 == pb.DEFAULT_MULTIPLIER & 1 for m in mults)


def test_genparams_validation():
    bad = [dict(n=10), dict(n=10, d=2, degrees=np.ones(10, dtype=np.uint64)), dict(n=5, d=0),
           dict(n=5, d=2, n0=6), dict(n=5, d=2, n0=-1),
           dict(n=5, d=2, n0=1, seed_edges=np.array([0, 1, 2], dtype=np.uint64)),
           dict(n=5, d=2, n0=1, seed_edges=np.array([0, 1], dtype=np.uint64)),
           dict(n=5, d=2, max_attempts=0), dict(n=2**58, d=1),
           dict(n=5, n0=1, degrees=np.array([2, 2], dtype=np.uint64)),
           dict(n=5, d=2, no_self_loops=True), dict(n=5, d=2, no_parallel_edges=True)]
    for kw in bad:
        with pytest.raises(pb.ParameterError):
            pb.GenParams(**kw)


def test_genparams_derived():
    p = pb.GenParams(n=10, d=2)
    assert (p.m0, p.m, pb.edge_count(p)) == (0, 20, 20)
    p = pb.GenParams(n=10, d=2, n0=3, seed_edges=TRIANGLE)
    assert (p.m0, p.m) == (3, 17) and p.degree_of(5) == 2
    assert p.first_edge_of(3) == 3 and p.first_edge_of(4) == 5
    for v in (2, 10):
        with pytest.raises(pb.ParameterError):
            p.degree_of(v)
    src = np.array([0, 1], dtype=np.int32)
    q = pb.GenParams(n=5, d=1, n0=2, seed_edges=src)
    src[0] = 99
    assert q.seed_edges.dtype == np.uint64 and q.seed_edges.tolist() == [0, 1]
    assert pb.GenParams(n=10**10, d=100).m == 10**12


def test_plan_batches_reference_cases():
    p = pb.GenParams(n=30, d=2)
    assert pb.plan_batches(p, 30) == [pb.Batch(0, 30), pb.Batch(30, 60)]
    assert pb.plan_batches(p, 25) == [pb.Batch(0, 25), pb.Batch(25, 50), pb.Batch(50, 60)]
    u = pb.GenParams(n=40, d=3, n0=3, seed_edges=TRIANGLE)
    assert pb.plan_batches(u, 1000) == [pb.Batch(3, 114)]
    q = pb.GenParams(n=30, d=4, n0=3, seed_edges=TRIANGLE)
    got = pb.plan_batches(q, 30, granularity=pb.Granularity.NODE)
    assert got[0] == pb.Batch(3, 31, pb.Granularity.NODE)
    with pytest.raises(pb.ParameterError):
        pb.plan_batches(u, 0)
    rng = np.random.default_rng(40)
    for _ in range(20):
        n0 = int(rng.integers(0, 4))
        seed = ring_edges(n0) if n0 else None
        p = pb.GenParams(n=int(rng.integers(n0 + 1, 80)), d=int(rng.integers(1, 6)), n0=n0, seed_edges=seed)
        pos = p.m0
        for b in pb.plan_batches(p, int(rng.integers(1, 40))):
            assert b.lo == pos and b.hi > b.lo
            pos = b.hi
        assert pos == p.m


def test_shard_range_exact_cover():
    rng = np.random.default_rng(3)
    for _ in range(200):
        lo = int(rng.integers(0, 10**12))
        hi = lo + int(rng.integers(0, 10**6))
        G = int(rng.integers(1, 9))
        pos = lo
        for g in range(G):
            a, b = pb.parallel.shard_range(lo, hi, g, G)
            assert a == pos and b >= a
            pos = b
        assert pos == hi
    assert pb.parallel.shard_range(0, 10**12, 7, 8) == (875 * 10**9, 10**12)
    with pytest.raises(pb.ParameterError):
        pb.parallel.shard_range(0, 10, 2, 2)


def test_run_validation():
    p = pb.GenParams(n=10, d=2)
    with pytest.raises(pb.ParameterError):
        pb.run(p, pb.DiscardConsumer(), workers=0)
    with pytest.raises(pb.ParameterError):
        pb.run(p, pb.DiscardConsumer(), batch_size=0)
    with pytest.raises(pb.ParameterError):
        pb.DegreeCountConsumer(-1)
    with pytest.raises(pb.ParameterError):
        pb.DegreeCounter.zeros(-1)


def test_count_edge_and_merge_semantics():
    c = pb.DegreeCounter.zeros(4)
    pb.count_edge(c, pb.Edge(0, 3))
    pb.count_edge(c, pb.Edge(3, 1))
    pb.count_edge(c, pb.Edge(1, 9))
    assert c.counts.tolist() == [1, 2, 0, 2]
    d = pb.DegreeCounter.zeros(2)
    pb.count_edge(d, pb.Edge(1, 1))
    assert d.counts.tolist() == [0, 2]
    a = pb.DegreeCounter(3, np.array([1, 0, 2], dtype=np.int64))
    b = pb.DegreeCounter(3, np.array([0, 5, 1], dtype=np.int64))
    assert pb.merge(a, b).counts.tolist() == [1, 5, 3]
    with pytest.raises(pb.ParameterError):
        pb.merge(a, pb.DegreeCounter.zeros(4))


def test_exponent_fit_on_synthetic_counts():
    """The tests' power-law estimator recovers a known exponent."""
    from powerlaw import mle_exponent

    rng = np.random.default_rng(11)
    gamma = 3.0
    # discrete power-law sample via inverse transform of the continuous law
    x = np.floor((16 - 0.5) * (1 - rng.random(200_000)) ** (-1 / (gamma - 1)) + 0.5).astype(np.int64)
    assert abs(mle_exponent(x, kmin=16) - gamma) < 0.05
    with pytest.raises(ValueError):
        mle_exponent(np.array([5] * 10), kmin=5)


def test_edge_file_writer_positional_semantics(tmp_path):
    # cli.py:121-145: edge i at byte offset 16*(i - m0), file pre-sized, LE u64
    path = tmp_path / "edges.bin"
    w = pb.EdgeFileWriter(str(path), 3, 10)
    ctx = w.new_context(0)
    ctx = w.accept_block(ctx, 8, np.array([[7, 1], [7, 2]], dtype=np.uint64))
    ctx = w.accept_block(ctx, 3, np.array([[3, 0]], dtype=np.uint64))
    w.close()
    assert w.merge([ctx]) == 48
    data = np.frombuffer(path.read_bytes(), dtype="<u8").reshape(-1, 2)
    assert data.shape == (10, 2)
    assert data[0].tolist() == [3, 0] and data[5].tolist() == [7, 1] and data[6].tolist() == [7, 2]
    assert (data[1:5] == 0).all()
    with pytest.raises(pb.ParameterError):
        pb.EdgeFileWriter(str(tmp_path / "x.bin"), 0, -1)


def test_degree_sequence_validation_and_host_planning():
    """build_prefix's checks (degreeseq.py:87-109) on the host; m, first
    edges and degrees of a degree-sequence family without touching a GPU."""
    for bad, msg in ((np.array([[1, 2]]), "one-dimensional"), (np.array([1.5]), "integers"),
                     (np.array([2, -1]), "non-negative"),
                     (np.array([2**63, 2**63], dtype=np.uint64), "overflows"),
                     (np.array([2**58], dtype=np.uint64), "maximum")):
        with pytest.raises(pb.ParameterError, match=msg):
            pb.degreeseq.validate_degrees(bad, 0, 0)
    with pytest.raises(pb.ParameterError, match="length"):
        pb.GenParams(n=5, n0=1, degrees=np.array([1, 2], dtype=np.uint64))
    p = pb.GenParams(n=6, n0=3, degrees=np.array([2, 0, 3], dtype=np.uint64), seed_edges=TRIANGLE)
    assert (p.m0, p.m) == (3, 8)
    assert [p.first_edge_of(v) for v in (3, 4, 5)] == [3, 5, 5]
    assert [p.degree_of(v) for v in (3, 4, 5)] == [2, 0, 3]
    with pytest.raises(pb.ParameterError):
        pb.GenParams(n=10, d=2).prefix


def test_node_aligned_cuts_and_shards():
    """Chunk cuts and rank shards land on node boundaries when an option
    flag makes generation node-granular (driver.py:131-158)."""
    from paper_1602_07106_b200 import generator as G, parallel as P

    rng = np.random.default_rng(8)
    deg = rng.integers(0, 9, size=400).astype(np.uint64)
    deg[0] = 1
    fams = [pb.GenParams(n=300, d=7, n0=3, seed_edges=TRIANGLE, no_self_loops=True),
            pb.GenParams(n=403, n0=3, degrees=deg, seed_edges=TRIANGLE, no_parallel_edges=True)]
    for p in fams:
        if p.d is not None:
            starts = {p.m0 + k * p.d for k in range(p.n - p.n0)} | {p.m}
        else:
            starts = set(int(x) for x in p._host_W())
        for chunk in (1, 5, 37, 1000, 10**6):
            cuts = G._cuts(p, p.m0, p.m, chunk)
            assert cuts[0] == p.m0 and cuts[-1] == p.m
            assert all(a < b for a, b in zip(cuts, cuts[1:]))
            assert set(cuts) <= starts
        for ws in range(1, 9):
            pos = p.m0
            for r in range(ws):
                a, b = P.shard_range_for(p, p.m0, p.m, r, ws)
                assert a == pos and b >= a and b in starts
                pos = b
            assert pos == p.m
    plain = pb.GenParams(n=300, d=7)
    assert G._cuts(plain, 5, 50, 10) == [5, 15, 25, 35, 45, 50]
    assert P.shard_range_for(plain, 0, 100, 1, 3) == P.shard_range(0, 100, 1, 3)


def test_crc_table_constant_matches_reference(golden):
    arrays, _ = golden
    assert np.array_equal(np.array(pb.CRC32C_TABLE, dtype=np.uint32), arrays["crc_table"])


def test_balanced_cuts():
    """parallel.balanced_cuts: equal-cost contiguous parts under the
    piecewise-constant density the measured step implies; a cover of the
    range with monotone, tile-aligned interior cuts."""
    from paper_1602_07106_b200 import parallel as P

    def cost(cuts, times, a, b):
        tot = 0.0
        for k in range(len(times)):
            lo, hi = max(a, cuts[k]), min(b, cuts[k + 1])
            if hi > lo:
                tot += times[k] * (hi - lo) / (cuts[k + 1] - cuts[k])
        return tot

    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(1, 9))
        lo = int(rng.integers(0, 1 << 20))
        hi = lo + int(rng.integers(n, 1 << 34))
        cuts = [P.shard_range(lo, hi, r, n)[0] for r in range(n)] + [hi]
        times = list(rng.uniform(0.5, 3.0, size=n))
        new = P.balanced_cuts(cuts, times, align=1)
        assert new[0] == lo and new[-1] == hi and all(x <= y for x, y in zip(new, new[1:]))
        parts = [cost(cuts, times, new[i], new[i + 1]) for i in range(n)]
        assert max(parts) - min(parts) <= 1e-6 * sum(times) + max(times) * n / max(1, hi - lo) * 4
        al = P.balanced_cuts(cuts, times)
        assert all(x % 256 == 0 for x in al[1:-1]) and al[0] == lo and al[-1] == hi
    assert P.balanced_cuts([0, 5, 10], [1.0, 1.0], align=1) == [0, 5, 10]
    assert P.balanced_cuts([0, 100, 200, 300, 400], [1, 1, 2, 4], align=1) == [0, 200, 300, 350, 400]
    with pytest.raises(pb.ParameterError):
        P.balanced_cuts([0, 1], [1.0, 2.0])


def test_routed_slice_nodes():
    """Owner slices of the routed full histogram: multiples of 2^16 (>= the
    57344 nodes one count CTA holds, so a CTA's nodes have at most two
    owners) that cover [0, n) with the last owner possibly short or empty."""
    for n in (1, 65_536, 65_537, 10**8, (1 << 25) + 12_345, (1 << 31) - 1):  # 2m < 2^32 bounds n
        for owners in (1, 2, 3, 8, 16):
            S = pb.parallel.routed_slice_nodes(n, owners)
            assert S % 65_536 == 0 and S >= 65_536 and S * owners >= n
            assert S - 65_536 < (n + owners - 1) // owners  # no more padding than one 2^16 block
            assert S < (1 << 32)
