"""GPU parity of the node-granular rows: f4 degree sequences
(device prefix / rank index, the three owner lookups, generation and degree
counts in the tile kernels) and f3 option flags (the node kernel), through
the C ABI, against fixtures made by the reference itself
(tests/golden/make_golden_nodes.py) and against the CPU oracle.

Bar: bit-exact edges, probe totals, counts and error messages."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import TRIANGLE
from test_oracle_nodes import oparams_deg, oparams_flag

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_1602_07106_b200")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _hc(kind: str, salt: int = 0):
    return pb.HashConfig(kind=pb.HashKind(kind), attempt_salt=salt)


def params_deg(c, arrays, **kw) -> "pb.GenParams":
    return pb.GenParams(n=c["n"], n0=c["n0"], degrees=arrays[f"{c['name']}_degrees"],
                        seed_edges=None if c["seed"] is None else np.array(c["seed"], dtype=np.uint64),
                        hash=_hc(c["kind"]), **kw)


def params_flag(c, arrays) -> "pb.GenParams":
    kw = dict(n=c["n"], n0=c["n0"], seed_edges=np.array(c["seed"], dtype=np.uint64),
              no_self_loops=c["nsl"], no_parallel_edges=c["npe"], hash=_hc(c["kind"], c["salt"]))
    if c["has_degrees"]:
        kw["degrees"] = arrays[f"{c['name']}_degrees"]
    else:
        kw["d"] = c["d"]
    return pb.GenParams(**kw)


# --------------------------------------------------------------------------- f4 index

def test_degree_index_vs_reference(golden_nodes):
    arrays, meta = golden_nodes
    g = meta["index"]
    pi = pb.build_prefix(arrays["index_degrees"], m0=g["m0"], n0=g["n0"])
    assert np.array_equal(pi.W, arrays["index_W"]) and pi.m == g["m"]
    rb = pb.build_rank_bits(pi)
    assert rb.n_ones == g["n_ones"] and rb.nbits == g["m"]
    assert np.array_equal(rb.words, arrays["index_words"])
    assert np.array_equal(pb.degreeseq.rank1_many(rb, arrays["index_es"]), arrays["index_rank1"])
    es, want = arrays["index_gen_es"], arrays["index_owner"]
    assert np.array_equal(pb.degreeseq.node_of_edge_many(es, rb), want)
    assert np.array_equal(pb.degreeseq.node_of_edge_bisect_many(es, pi), want)
    assert np.array_equal(pb.degreeseq.owners_of_edges_deferred(es, pi), want)
    if g["owners"] is not None:
        assert [int(x) for x in rb.owners[:8]] == g["owners"]


def test_degree_index_reference_unit_cases():
    # reference tests/test_degreeseq.py:40-178 restated
    pi = pb.build_prefix(np.array([3, 1, 2], dtype=np.uint64), m0=0, n0=0)
    assert pi.W.tolist() == [0, 3, 4] and pi.m == 6 and pi.n_nodes == 3
    rb = pb.build_rank_bits(pb.build_prefix(np.array([1, 2, 1], dtype=np.uint64), m0=0, n0=0))
    assert rb.nbits == 4 and int(rb.words[0]) == 0b1011 and rb.n_ones == 3 and rb.owners is None
    assert [pb.degreeseq.rank1(rb, e) for e in range(4)] == [1, 2, 2, 3]
    rb = pb.build_rank_bits(pb.build_prefix(np.array([2, 2], dtype=np.uint64), m0=2, n0=2))
    assert rb.nbits == 6 and int(rb.words[0]) == (1 << 2) | (1 << 4)
    rb = pb.build_rank_bits(pb.build_prefix(np.array([], dtype=np.uint64), m0=0, n0=0))
    assert rb.nbits == 0 and rb.n_ones == 0
    pi = pb.build_prefix(np.array([2, 0, 3], dtype=np.uint64), m0=0, n0=0)
    rb = pb.build_rank_bits(pi)
    assert rb.owners is not None
    assert [pb.node_of_edge(e, rb) for e in range(5)] == [0, 0, 2, 2, 2]
    assert [pb.node_of_edge_bisect(e, pi) for e in range(5)] == [0, 0, 2, 2, 2]
    pi = pb.build_prefix(np.array([2], dtype=np.uint64), m0=3, n0=1)
    rb = pb.build_rank_bits(pi)
    for bad in (2, 5):
        with pytest.raises(pb.ParameterError):
            pb.node_of_edge(bad, rb)
        with pytest.raises(pb.ParameterError):
            pb.node_of_edge_bisect(bad, pi)
    with pytest.raises(pb.ParameterError):
        pb.degreeseq.rank1(rb, 5)
    pi = pb.build_prefix(np.array([3, 1, 2], dtype=np.uint64), m0=0, n0=0)
    assert pb.resolve_targets_deferred([(4, 6)], pi) == [(2, 1)]
    assert pb.resolve_targets_deferred([], pi) == []
    with pytest.raises(pb.ParameterError):
        pb.resolve_targets_deferred([(0, 3)], pi)
    assert [pb.first_half_pos(v, pi) for v in range(3)] == [0, 6, 8]
    for bad in (np.array([[1]]), np.array([1.5]), np.array([-1, 2])):
        with pytest.raises(pb.ParameterError):
            pb.build_prefix(bad, m0=0, n0=0)
    with pytest.raises(pb.ParameterError):
        pb.build_prefix(np.array([2**63, 2**63], dtype=np.uint64), m0=0, n0=0)


def test_degree_index_random_agreement_and_uniform_reduction():
    rng = np.random.default_rng(13)
    for trial in range(6):
        n_nodes = int(rng.integers(1, 200_000))
        deg = rng.integers(0, 7, size=n_nodes).astype(np.uint64)
        deg[0] = max(int(deg[0]), 1)
        m0, n0 = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        pi = pb.build_prefix(deg, m0=m0, n0=n0)
        rb = pb.build_rank_bits(pi)
        es = rng.integers(pi.m0, pi.m, size=50_000, dtype=np.uint64)
        W = pi.W
        want = (np.searchsorted(W, es, side="right") - 1 + n0).astype(np.uint64)
        assert np.array_equal(pb.degreeseq.node_of_edge_many(es, rb), want)
        assert np.array_equal(pb.degreeseq.node_of_edge_bisect_many(es, pi), want)
        assert np.array_equal(pb.degreeseq.owners_of_edges_deferred(es, pi), want)
    d, m0, n0, n = 4, 3, 3, 40
    pi = pb.build_prefix(np.full(n - n0, d, dtype=np.uint64), m0=m0, n0=n0)
    es = np.arange(m0, pi.m, dtype=np.uint64)
    assert np.array_equal(pb.degreeseq.node_of_edge_many(es, pb.build_rank_bits(pi)),
                          (es - np.uint64(m0)) // np.uint64(d) + np.uint64(n0))


# --------------------------------------------------------------------------- f4 generation

def test_degree_sequence_blocks_vs_reference(golden_nodes):
    arrays, meta = golden_nodes
    for c in meta["degseq"]:
        p = params_deg(c, arrays)
        assert p.m == c["m"]
        for res in ("rank", "bisect", "deferred"):
            got, probes = pb.generate_block(p.m0, p.m, p, resolution=res)
            assert _sha(got) == c["sha256"] and probes == c["probes"], (c["name"], res)
        lo, hi, sub_sha, sub_pr = c["sub"]
        sub, sp = pb.generate_block(lo, hi, p)
        assert _sha(sub) == sub_sha and sp == sub_pr, c["name"]
    with pytest.raises(pb.ParameterError, match="unknown resolution"):
        pb.generate_block(0, 1, params_deg(meta["degseq"][0], arrays), resolution="sideways")


def test_degree_sequence_counts_vs_reference(golden_nodes):
    arrays, meta = golden_nodes
    for c in meta["counts"]:
        case = next(x for x in meta["degseq"] if x["name"] == c["case"])
        p = params_deg(case, arrays)
        counter, stats = pb.degree_counts(p, K=c["K"]) if c["K"] else pb.degree_counts(p)
        assert _sha(counter.counts) == c["sha256"] and stats.hash_probes == c["probes"], c


def test_degree_sequence_edges_at_and_node_edges(golden_nodes):
    arrays, meta = golden_nodes
    c = meta["degseq"][5]
    p = params_deg(c, arrays)
    full = arrays[f"{c['name']}_edges"]
    ids = np.arange(p.m0, p.m, 7, dtype=np.uint64)
    e, _ = pb.edges_at(ids, p)
    assert np.array_equal(e, full[(ids - np.uint64(p.m0)).astype(np.int64)])
    for v in (p.n0, p.n0 + 3, p.n - 1):
        first, dv = p.first_edge_of(v), p.degree_of(v)
        got = pb.generate_node_edges(v, p)
        assert [tuple(x) for x in got] == [tuple(map(int, r)) for r in full[first - p.m0: first - p.m0 + dv]]


def test_degree_sequence_large_vs_oracle():
    """A million-node power-law-like sequence (zeros included): random
    unaligned subranges bit-exact vs the oracle, full window counts sum."""
    rng = np.random.default_rng(77)
    n_nodes = 10**6
    deg = np.minimum(rng.zipf(2.2, size=n_nodes), 500).astype(np.uint64)
    deg[rng.random(n_nodes) < 0.05] = 0
    deg[0] = 2
    p = pb.GenParams(n=3 + n_nodes, n0=3, degrees=deg, seed_edges=TRIANGLE)
    op = O.OParams(n=p.n, d=None, n0=3, seed_edges=tuple(int(x) for x in TRIANGLE),
                   degrees=tuple(int(x) for x in deg))
    for _ in range(4):
        lo = int(rng.integers(p.m0, p.m - 20000))
        hi = lo + int(rng.integers(1, 20000))
        got, pr = pb.generate_block(lo, hi, p)
        want, wp = O.generate_block(op, lo, hi)
        assert np.array_equal(got, want) and pr == wp
    counter, stats = pb.degree_counts(p)
    assert int(counter.counts.sum()) == 2 * p.m
    assert np.array_equal(counter.counts[3:] >= deg.astype(np.int64), np.ones(n_nodes, dtype=bool))
    K = 1000
    win, _ = pb.degree_counts(p, K=K)
    assert np.array_equal(win.counts, counter.counts[:K])


# --------------------------------------------------------------------------- f3 option flags

def test_option_flag_blocks_vs_reference(golden_nodes):
    arrays, meta = golden_nodes
    for c in meta["flags"]:
        p = params_flag(c, arrays)
        got, probes = pb.generate_block(p.m0, p.m, p)
        assert _sha(got) == c["sha256"] and probes == c["probes"], c["name"]
        lo, hi, sub_sha, sub_pr = c["sub"]
        sub, sp = pb.generate_block(lo, hi, p)
        assert _sha(sub) == sub_sha and sp == sub_pr, c["name"]
        counter, stats = pb.degree_counts(p)
        assert _sha(counter.counts) == c["counts_sha256"] and stats.hash_probes == c["counts_probes"], c["name"]
        if c["nsl"]:
            assert (got[:, 1] < got[:, 0]).all()
        if c["npe"] and not c["has_degrees"]:
            t = np.sort(got[:, 1].reshape(-1, c["d"]), axis=1)
            assert (np.diff(t, axis=1) != 0).all()


def test_option_flag_errors_match_reference(golden_nodes):
    _, meta = golden_nodes
    for c in meta["infeasible"]:
        p = pb.GenParams(n=c["n"], d=c["d"], n0=c["n0"], seed_edges=np.array(c["seed"], dtype=np.uint64),
                         no_self_loops=True, no_parallel_edges=True, max_attempts=c["max_attempts"])
        with pytest.raises(pb.InfeasibleTargetsError) as ei:
            pb.generate_block(p.m0, p.m, p)
        assert str(ei.value) == c["message"]
        with pytest.raises(pb.InfeasibleTargetsError, match="node 2"):
            pb.generate_node_edges(2, p)
    p = pb.GenParams(n=40, d=3, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    with pytest.raises(pb.ParameterError, match="node boundary"):
        pb.generate_block(4, p.m, p)
    with pytest.raises(pb.ParameterError, match="node boundary"):
        pb.generate_block(p.m0, p.m - 1, p)
    with pytest.raises(pb.ParameterError):
        pb.generate_edge(5, p)
    with pytest.raises(pb.ParameterError):
        pb.edges_at([5], p)


def test_option_flags_node_edges_and_chain_sharing():
    p = pb.GenParams(n=30, d=4, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    for v in (3, 17, 29):
        assert len({e.target for e in pb.generate_node_edges(v, p)}) == 1
    q = pb.GenParams(n=40, d=3, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    block, _ = pb.generate_block(q.m0, q.m, q)
    want = [tuple(e) for v in range(3, 40) for e in pb.generate_node_edges(v, q)]
    assert [tuple(map(int, r)) for r in block] == want


def test_option_flags_large_vs_oracle_and_chunked(monkeypatch, tmp_path):
    """1e5-node runs bit-exact vs the oracle; node-aligned host chunks, the
    binary writer and world-size-independent counts on the flag path."""
    from paper_1602_07106_b200 import generator as G, io as IO

    seed = np.array([x for u in range(6) for v in range(u + 1, 6) for x in (u, v)], dtype=np.uint64)
    for nsl, npe in ((True, False), (False, True), (True, True)):
        p = pb.GenParams(n=10**5, d=4, n0=6, seed_edges=seed, no_self_loops=nsl, no_parallel_edges=npe)
        op = O.OParams(n=p.n, d=4, n0=6, seed_edges=tuple(int(x) for x in seed), no_self_loops=nsl,
                       no_parallel_edges=npe)
        want, wp = O.generate_block(op, p.m0, p.m)
        got, pr = pb.generate_block(p.m0, p.m, p)
        assert np.array_equal(got, want) and pr == wp
        monkeypatch.setattr(G, "HOST_CHUNK_EDGES", 4097)
        got2, pr2 = pb.generate_block(p.m0, p.m, p)
        assert np.array_equal(got2, want) and pr2 == wp
        monkeypatch.setattr(IO, "FILE_CHUNK_EDGES", 10001)
        path = tmp_path / f"f{int(nsl)}{int(npe)}.bin"
        nbytes, _ = pb.write_edges_binary(str(path), p)
        assert nbytes == 16 * (p.m - p.m0)
        assert np.array_equal(np.fromfile(path, dtype="<u8").reshape(-1, 2), want)
        counts = np.zeros(p.n, dtype=np.int64)
        O.count_block(counts, want)
        counts += np.bincount(seed.astype(np.int64), minlength=p.n)
        counter, _ = pb.degree_counts(p)
        assert np.array_equal(counter.counts, counts)


def test_option_flags_with_degree_sequence_vs_oracle():
    rng = np.random.default_rng(5)
    deg = rng.integers(0, 9, size=50_000).astype(np.uint64)
    deg[0] = 3
    seed = np.array([x for u in range(7) for v in range(u + 1, 7) for x in (u, v)], dtype=np.uint64)
    for kind in ("crc", "simple"):
        p = pb.GenParams(n=7 + deg.size, n0=7, degrees=deg, seed_edges=seed, no_self_loops=True,
                         no_parallel_edges=True, hash=_hc(kind))
        op = O.OParams(n=p.n, d=None, n0=7, seed_edges=tuple(int(x) for x in seed),
                       kind=O.KIND_CRC if kind == "crc" else O.KIND_SIMPLE, degrees=tuple(int(x) for x in deg),
                       no_self_loops=True, no_parallel_edges=True)
        want, wp = O.generate_block(op, p.m0, p.m)
        got, pr = pb.generate_block(p.m0, p.m, p)
        assert np.array_equal(got, want) and pr == wp
        v = 7 + 1234
        lo = p.first_edge_of(v)
        hi = p.first_edge_of(v + 500)
        sub, sp = pb.generate_block(lo, hi, p)
        assert np.array_equal(sub, want[lo - p.m0: hi - p.m0])


def test_degree_count_windows_edge_cases_vs_oracle():
    """K in {0, 1, n0, n0+1, n, n+17} for uniform, degree-sequence and
    flagged families, counts of subranges with the seed folded in; the
    device window / full kernels (and the flag path's chunked counts) must
    equal count_block over the oracle's edges."""
    rng = np.random.default_rng(31)
    deg = rng.integers(0, 6, size=4000).astype(np.uint64)
    deg[0] = 2
    seed = np.array([x for u in range(5) for v in range(u + 1, 5) for x in (u, v)], dtype=np.uint64)
    fams = [
        (pb.GenParams(n=5000, d=3, n0=5, seed_edges=seed),
         O.OParams(n=5000, d=3, n0=5, seed_edges=tuple(int(x) for x in seed))),
        (pb.GenParams(n=4005, n0=5, degrees=deg, seed_edges=seed),
         O.OParams(n=4005, d=None, n0=5, seed_edges=tuple(int(x) for x in seed), degrees=tuple(int(x) for x in deg))),
        (pb.GenParams(n=3000, d=4, n0=5, seed_edges=seed, no_self_loops=True, no_parallel_edges=True),
         O.OParams(n=3000, d=4, n0=5, seed_edges=tuple(int(x) for x in seed), no_self_loops=True,
                   no_parallel_edges=True)),
    ]
    for p, op in fams:
        want_edges, _ = O.generate_block(op, op.m0, op.m)
        for K in (0, 1, p.n0, p.n0 + 1, p.n, p.n + 17):
            want = np.zeros(K, dtype=np.int64)
            O.count_block(want, want_edges)
            O.count_block(want, np.asarray(seed, dtype=np.uint64))
            counter, _ = pb.degree_counts(p, K=K)
            assert counter.K == K and np.array_equal(counter.counts, want), (p, K)


def test_degree_sequence_rank_path_without_dense_map(golden_nodes, monkeypatch):
    """The generator uses the dense owner map when it fits; with the map
    disabled the rank-directory lookups must give the same bytes."""
    from paper_1602_07106_b200 import generator as G

    arrays, meta = golden_nodes
    monkeypatch.setattr(G, "DENSE_OWNER_MAX_BYTES", 0)
    for c in meta["degseq"][::5]:
        p = params_deg(c, arrays)
        assert p._index()[2] is None
        got, probes = pb.generate_block(p.m0, p.m, p)
        assert _sha(got) == c["sha256"] and probes == c["probes"], c["name"]
    for c in meta["counts"]:
        case = next(x for x in meta["degseq"] if x["name"] == c["case"])
        p = params_deg(case, arrays)
        counter, stats = pb.degree_counts(p, K=c["K"]) if c["K"] else pb.degree_counts(p)
        assert _sha(counter.counts) == c["sha256"], c


def test_no_parallel_edges_high_degree_nodes_vs_oracle():
    """Nodes above the hash-set threshold (degree > 64) run node_big_kernel:
    uniform d = 300 and power-law degree sequences with hubs, with and
    without no_self_loops, bit-exact (edges and probe totals) vs the oracle."""
    seed = np.array([x for u in range(320) for v in range(u + 1, 320) for x in (u, v)], dtype=np.uint64)
    s_t = tuple(int(x) for x in seed)
    for nsl in (False, True):
        p = pb.GenParams(n=2000, d=300, n0=320, seed_edges=seed, no_self_loops=nsl, no_parallel_edges=True)
        op = O.OParams(n=2000, d=300, n0=320, seed_edges=s_t, no_self_loops=nsl, no_parallel_edges=True)
        got, pr = pb.generate_block(p.m0, p.m, p)
        want, wp = O.generate_block(op, op.m0, op.m)
        assert np.array_equal(got, want) and pr == wp, ("uniform", nsl)
    rng = np.random.default_rng(3)
    deg = np.sort(np.minimum(rng.zipf(2.0, size=20000) + 1, 700)).astype(np.uint64)  # hubs late
    for nsl in (False, True):
        p = pb.GenParams(n=320 + deg.size, n0=320, degrees=deg, seed_edges=seed, no_self_loops=nsl,
                         no_parallel_edges=True)
        op = O.OParams(n=p.n, d=None, n0=320, seed_edges=s_t, degrees=tuple(int(x) for x in deg),
                       no_self_loops=nsl, no_parallel_edges=True)
        got, pr = pb.generate_block(p.m0, p.m, p)
        want, wp = O.generate_block(op, op.m0, op.m)
        assert np.array_equal(got, want) and pr == wp, ("degrees", nsl)
        t = got[:, 1]
        for v in (p.n - 1, p.n - 2):  # the hubs: distinct targets
            a, b = p.first_edge_of(v) - p.m0, p.first_edge_of(v) - p.m0 + p.degree_of(v)
            assert len(set(t[a:b].tolist())) == b - a
        # degree counts through the flag path's chunked generate + count
        want_c = np.zeros(p.n, dtype=np.int64)
        O.count_block(want_c, want)
        O.count_block(want_c, seed)
        counter, st = pb.degree_counts(p)
        assert np.array_equal(counter.counts, want_c) and st.hash_probes == wp


def test_no_self_loops_fused_counts_match_generated_edges():
    """no_self_loops alone counts per node (node_count_kernel: dv added to the
    node and to its one target) instead of materialising edge rows; windows
    and full counts equal the histogram of the generated edges, probes too."""
    rng = np.random.default_rng(77)
    deg = rng.integers(0, 9, size=30_000).astype(np.uint64)
    for p in (pb.GenParams(n=50_000, d=6, n0=3, seed_edges=TRIANGLE, no_self_loops=True),
              pb.GenParams(n=3 + deg.size, n0=3, degrees=deg, seed_edges=TRIANGLE, no_self_loops=True)):
        edges, probes = pb.generate_block(p.m0, p.m, p)
        seed_hist = np.bincount(np.asarray(p.seed_edges, dtype=np.int64), minlength=p.n)
        full = np.bincount(edges.astype(np.int64).ravel(), minlength=p.n) + seed_hist
        for K in (p.n, 1000, 1):
            counter, stats = pb.degree_counts(p, K=K) if K != p.n else pb.degree_counts(p)
            assert np.array_equal(counter.counts, full[:K]) and stats.hash_probes == probes, K


@pytest.mark.parametrize("K", [None, 4000])
def test_no_parallel_edges_counts_partitioned_equals_direct(K, monkeypatch):
    """no_parallel_edges counts from the materialised edge rows: targets
    through the partitioned pass (rows_targets_kernel + scatter + slice
    counts), sources per node, equal to the direct count_pairs_kernel."""
    deg = np.random.default_rng(5).integers(0, 7, size=40_000).astype(np.uint64)
    seed = np.array([x for a in range(8) for b in range(a + 1, 8) for x in (a, b)], dtype=np.uint64)
    for p in (pb.GenParams(n=60_000, d=5, n0=8, seed_edges=seed, no_parallel_edges=True),
              pb.GenParams(n=8 + deg.size, n0=8, degrees=deg, seed_edges=seed, no_parallel_edges=True,
                           no_self_loops=True)):
        kk = p.n if K is None else K
        got = {}
        for mode in ("partition", "direct"):
            monkeypatch.setenv("PARBA_FULL_MODE", mode)
            counter, stats = pb.degree_counts(p, K=kk) if K else pb.degree_counts(p)
            got[mode] = (counter.counts.copy(), stats.hash_probes)
        assert np.array_equal(got["partition"][0], got["direct"][0])
        assert got["partition"][1] == got["direct"][1]


def test_flag_counts_small_chunks_equal_one_chunk(monkeypatch):
    """Option-flag counts cut into many node-aligned chunks (degree sequence:
    chunk bounds by edge lower bounds in W, zero-degree nodes included) equal
    the single-chunk counts, probes included."""
    deg = np.random.default_rng(11).integers(0, 9, size=20_000).astype(np.uint64)
    deg[::7] = 0
    seed = np.array([x for a in range(9) for b in range(a + 1, 9) for x in (a, b)], dtype=np.uint64)
    for p in (pb.GenParams(n=9 + deg.size, n0=9, degrees=deg, seed_edges=seed, no_parallel_edges=True),
              pb.GenParams(n=20_000, d=7, n0=9, seed_edges=seed, no_parallel_edges=True, no_self_loops=True)):
        whole, wp = pb.degree_counts(p)
        monkeypatch.setenv("PARBA_COUNT_CHUNK_EDGES", "1001")
        parts, pp = pb.degree_counts(p)
        monkeypatch.delenv("PARBA_COUNT_CHUNK_EDGES")
        assert np.array_equal(whole.counts, parts.counts) and wp.hash_probes == pp.hash_probes


def test_option_flags_reject_beyond_2p51_edges():
    # the node kernels' FP64 remainder needs chain values < 2^52: m <= 2^51
    p = pb.GenParams(n=1 << 40, d=1 << 12, n0=3, seed_edges=TRIANGLE, no_self_loops=True)
    assert p.m > 1 << 51
    lo = p.m0 + (p.n - p.n0 - 1) * p.d
    with pytest.raises(pb.ParameterError, match="2\\^51"):
        pb.generate_block(lo, lo + p.d, p)


def test_degree_sequence_full_counts_by_position(monkeypatch):
    """Degree-sequence full histograms through the opt-in position pass (targets
    partitioned as positions, owners resolved in order from the dense map,
    seed-graph targets counted directly) equal the owner-partitioned pass and
    the direct kernel, probes included; zero degrees and hubs included."""
    rng = np.random.default_rng(31)
    deg = np.minimum(rng.zipf(2.0, size=300_000) + rng.integers(0, 3, size=300_000), 5000).astype(np.uint64)
    deg[::11] = 0
    p = pb.GenParams(n=3 + deg.size, n0=3, degrees=deg, seed_edges=TRIANGLE)
    assert p._index()[2] is not None  # the dense owner map exists
    got = {}
    for name, mode, pos in (("pos", "partition", "1"), ("owner", "partition", "0"), ("direct", "direct", "0")):
        monkeypatch.setenv("PARBA_FULL_MODE", mode)
        monkeypatch.setenv("PARBA_POS_MODE", pos)
        counter, stats = pb.degree_counts(p)
        got[name] = (counter.counts.copy(), stats.hash_probes)
    for name in ("owner", "direct"):
        assert np.array_equal(got["pos"][0], got[name][0]) and got["pos"][1] == got[name][1], name
    assert int(got["pos"][0].sum()) == 2 * p.m


@pytest.mark.parametrize("d", [1, 3, 33, 300])
def test_no_self_loops_warp_rows_vs_oracle(d):
    """no_self_loops alone with uniform d runs node_nsl_kernel (one chain per
    node, the warp's rows stored cooperatively); node ranges that start and
    end off a 32-node boundary, bit-exact with probes vs the oracle."""
    k = 5
    seed = np.array([x for a in range(k) for b in range(a + 1, k) for x in (a, b)], dtype=np.uint64)
    p = pb.GenParams(n=3000 + 77, d=d, n0=k, seed_edges=seed, no_self_loops=True)
    op = O.OParams(n=p.n, d=d, n0=k, seed_edges=tuple(int(x) for x in seed), no_self_loops=True)
    for lo_node, hi_node in ((k, p.n), (k + 13, p.n - 7), (k + 40, k + 41)):
        lo, hi = p.m0 + (lo_node - k) * d, p.m0 + (hi_node - k) * d
        got, pr = pb.generate_block(lo, hi, p)
        want, wp = O.generate_block(op, lo, hi)
        assert np.array_equal(got, want) and pr == wp, (lo_node, hi_node)


def test_no_self_loops_degree_sequence_warp_rows_vs_oracle():
    """node_nsl_kernel on a degree sequence (zeros, hubs, runs of zero-degree
    nodes, ragged node ranges): rows mapped to nodes by the warp's degree
    prefix, bit-exact with probes vs the oracle."""
    rng = np.random.default_rng(17)
    deg = np.minimum(rng.zipf(1.8, size=4000), 700).astype(np.uint64)
    deg[::5] = 0
    deg[100:170] = 0  # a whole warp of zero-degree nodes
    k = 6
    seed = np.array([x for a in range(k) for b in range(a + 1, k) for x in (a, b)], dtype=np.uint64)
    p = pb.GenParams(n=k + deg.size, n0=k, degrees=deg, seed_edges=seed, no_self_loops=True)
    op = O.OParams(n=p.n, d=None, n0=k, seed_edges=tuple(int(x) for x in seed),
                   degrees=tuple(int(x) for x in deg), no_self_loops=True)
    W = np.concatenate([[p.m0], p.m0 + np.cumsum(deg.astype(np.int64))])
    for a, b in ((0, deg.size), (33, deg.size - 9), (101, 168), (7, 8)):
        lo, hi = int(W[a]), int(W[b])
        got, pr = pb.generate_block(lo, hi, p)
        want, wp = O.generate_block(op, lo, hi)
        assert np.array_equal(got, want) and pr == wp, (a, b)
