"""Property tests (hypothesis) of the host-side planning logic: batch plans,
rank shards and chunk cuts cover [m0, m) exactly once, in order, on node
boundaries whenever an option flag makes generation node-granular
(driver.py:131-158 semantics).  CPU only."""

from __future__ import annotations

import numpy as np
from hypothesis import given, settings, strategies as st

import paper_1602_07106_b200 as pb
from paper_1602_07106_b200 import generator as G, parallel as P


def _family(draw_deg, n0, d, flags, degrees):
    seed = np.array([x for i in range(n0) for x in (i, (i + 1) % n0)], dtype=np.uint64) if n0 else None
    kw = dict(n0=n0, seed_edges=seed, no_self_loops=flags and n0 > 0, no_parallel_edges=False)
    if draw_deg:
        deg = np.array(degrees, dtype=np.uint64)
        if deg.sum() == 0:
            deg[0] = 1
        return pb.GenParams(n=n0 + deg.size, degrees=deg, **kw)
    return pb.GenParams(n=n0 + len(degrees), d=d, **kw)


def _starts(p):
    if p.d is not None:
        return {p.m0 + k * p.d for k in range(p.n - p.n0)} | {p.m}
    return set(int(x) for x in p._host_W())


families = st.builds(
    _family,
    st.booleans(),
    st.integers(0, 4),
    st.integers(1, 9),
    st.booleans(),
    st.lists(st.integers(0, 7), min_size=1, max_size=300),
)


@settings(max_examples=150, deadline=None)
@given(p=families, batch=st.integers(1, 500))
def test_plan_batches_cover_exactly_once(p, batch):
    pos = p.m0
    starts = _starts(p)
    node = p.no_self_loops or p.no_parallel_edges
    for b in pb.plan_batches(p, batch):
        assert b.lo == pos and b.hi > b.lo
        if node:
            assert b.lo in starts and b.hi in starts
        pos = b.hi
    assert pos == p.m


@settings(max_examples=150, deadline=None)
@given(p=families, chunk=st.integers(1, 400), ws=st.integers(1, 9))
def test_cuts_and_shards_cover_exactly_once(p, chunk, ws):
    starts = _starts(p)
    node = p.has_flags
    cuts = G._cuts(p, p.m0, p.m, chunk)
    assert cuts[0] == p.m0 and cuts[-1] == p.m
    assert all(a < b for a, b in zip(cuts, cuts[1:])) or p.m == p.m0
    if node:
        assert set(cuts) <= starts
    pos = p.m0
    for r in range(ws):
        a, b = P.shard_range_for(p, p.m0, p.m, r, ws)
        assert a == pos and b >= a
        if node:
            assert a in starts and b in starts
        pos = b
    assert pos == p.m


@settings(max_examples=100, deadline=None)
@given(degrees=st.lists(st.integers(0, 50), max_size=200), m0=st.integers(0, 5), n0=st.integers(0, 5))
def test_degree_validation_total(degrees, m0, n0):
    deg, m = pb.degreeseq.validate_degrees(np.array(degrees, dtype=np.int64), m0, n0)
    assert deg.dtype == np.uint64 and m == m0 + sum(degrees)
