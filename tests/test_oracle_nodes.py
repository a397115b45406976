"""Pin the oracle's node-granular rows (f3 option flags, f4
degree sequences) against fixtures made by running the reference itself
(tests/golden/make_golden_nodes.py): full edge arrays / sha256 digests and
probe totals of generate_block, node-aligned interior blocks, and the
InfeasibleTargetsError cases."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle as O


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def oparams_deg(c, arrays) -> O.OParams:
    return O.OParams(n=c["n"], d=None, n0=c["n0"], seed_edges=tuple(c["seed"] or ()),
                     kind=O.KIND_CRC if c["kind"] == "crc" else O.KIND_SIMPLE,
                     degrees=tuple(int(x) for x in arrays[f"{c['name']}_degrees"]))


def oparams_flag(c, arrays) -> O.OParams:
    deg = tuple(int(x) for x in arrays[f"{c['name']}_degrees"]) if c["has_degrees"] else None
    return O.OParams(n=c["n"], d=None if deg else c["d"], n0=c["n0"], seed_edges=tuple(c["seed"]),
                     kind=O.KIND_CRC if c["kind"] == "crc" else O.KIND_SIMPLE, salt=c["salt"],
                     degrees=deg, no_self_loops=c["nsl"], no_parallel_edges=c["npe"])


def test_degree_sequences_vs_reference(golden_nodes):
    arrays, meta = golden_nodes
    for c in meta["degseq"]:
        p = oparams_deg(c, arrays)
        assert p.m == c["m"]
        got, probes = O.generate_block(p, p.m0, p.m)
        assert _sha(got) == c["sha256"] and probes == c["probes"], c["name"]
        if f"{c['name']}_edges" in arrays.files:
            assert np.array_equal(got, arrays[f"{c['name']}_edges"])
        lo, hi, sub_sha, sub_pr = c["sub"]
        sub, sp = O.generate_block(p, lo, hi)
        assert _sha(sub) == sub_sha and sp == sub_pr


def test_option_flags_vs_reference(golden_nodes):
    arrays, meta = golden_nodes
    for c in meta["flags"]:
        p = oparams_flag(c, arrays)
        got, probes = O.generate_block(p, p.m0, p.m)
        assert _sha(got) == c["sha256"] and probes == c["probes"], c["name"]
        lo, hi, sub_sha, sub_pr = c["sub"]
        sub, sp = O.generate_block(p, lo, hi)
        assert _sha(sub) == sub_sha and sp == sub_pr, c["name"]
        if c["nsl"]:
            assert (got[:, 1] < got[:, 0]).all()


def test_option_flags_node_boundaries_and_infeasible(golden_nodes):
    _, meta = golden_nodes
    p = O.OParams(n=40, d=3, n0=3, seed_edges=(0, 1, 1, 2, 2, 0), no_self_loops=True)
    with pytest.raises(O.NotNodeBoundary):
        O.generate_block(p, 4, p.m)
    with pytest.raises(O.NotNodeBoundary):
        O.generate_block(p, p.m0, p.m - 1)
    for c in meta["infeasible"]:
        q = O.OParams(n=c["n"], d=c["d"], n0=c["n0"], seed_edges=tuple(c["seed"]), no_self_loops=True,
                      no_parallel_edges=True, max_attempts=c["max_attempts"])
        with pytest.raises(O.Infeasible) as ei:
            O.generate_block(q, q.m0, q.m)
        assert c["message"].startswith(f"edge {ei.value.edge} of node")
