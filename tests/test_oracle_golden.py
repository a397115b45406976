"""Pin the CPU oracle (oracle/parba_oracle.c) before trusting it.

Every oracle function is checked against (a) the reference's own golden
vectors and frozen values (reference pkg/tests/helpers.py:11-18,
test_hashing.py:106-178, test_generator.py:43-45, 206-207) and (b) fixtures
produced by running the reference package itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN_CRC_N10_D2, GOLDEN_SIMPLE_N10_D2, RING10, TRIANGLE


def _cfg_params(c, n=10, d=1, n0=0, seed=()):
    kind, s0, s1, salt, mult = c
    return O.OParams(n=n, d=d, n0=n0, seed_edges=tuple(int(x) for x in seed),
                     kind=O.KIND_CRC if kind == "crc" else O.KIND_SIMPLE,
                     seed0=s0, seed1=s1, salt=salt, multiplier=mult)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _bitwise_crc(seed: int, word: int) -> int:
    crc = seed
    for k in range(64):
        bit = (crc ^ (word >> k)) & 1
        crc = (crc >> 1) ^ (0x82F63B78 * bit)
    return crc


def test_crc_table_matches_reference(golden):
    arrays, _ = golden
    assert np.array_equal(O.crc32c_table(), arrays["crc_table"])


def test_crc_known_answers():
    # reference test_hashing.py:106-115 (RFC 3720 through an inversion wrapper; raw accumulator)
    def standard(data: bytes) -> int:
        acc = 0xFFFFFFFF
        for off in range(0, len(data), 8):
            acc = O.crc32c_u64(acc, int.from_bytes(data[off:off + 8], "little"))
        return acc ^ 0xFFFFFFFF

    assert standard(b"\x00" * 32) == 0x8A9136AA
    assert standard(b"\xff" * 32) == 0x62A8AB43
    assert standard(bytes(range(32))) == 0x46DD794E
    assert O.crc32c_u64(0, 0) == 0
    assert O.crc32c_u64(0xFFFFFFFF, 0) == 0x73D74D75


def test_crc_fixture_and_bitwise(golden):
    arrays, _ = golden
    for s, w, want in zip(arrays["crc_seeds"], arrays["crc_words"], arrays["crc_out"]):
        got = O.crc32c_u64(int(s), int(w))
        assert got == int(want)
        assert got == _bitwise_crc(int(s), int(w))


def test_hash_frozen_values():
    # reference test_hashing.py:144-157, 175-178
    assert O.h_simple(3) == 1 and O.h_simple(11) == 9
    assert O.h_simple(2**32) == 2721204694 and O.h_simple(10**6) == 79004
    assert O.h_crc(3) == 2 and O.h_crc(1000) == 10 and O.h_crc(10**6) == 592013
    assert O.h_crc(1000, 7, 9) == 96
    assert O.h_crc(1) == 0 and O.h_simple(1) == 0


def test_hash_fixture_all_families(golden):
    arrays, meta = golden
    rs = arrays["hash_r"]
    for k, c in enumerate(meta["cfgs"]):
        p = _cfg_params(c)
        got = O.hash_many(p, rs)
        assert np.array_equal(got, arrays[f"hash_out_{k}"]), f"cfg {c}"


def test_chain_fixture(golden):
    arrays, meta = golden
    r0 = arrays["chain_r0"]
    for k, c in enumerate(meta["cfgs"]):
        p = _cfg_params(c)
        for stop in (0, 6, 1000):
            vals, probes = O.resolve_chain_block(p, r0, stop)
            assert np.array_equal(vals, arrays[f"chain_out_{k}_{stop}"])
            assert probes == meta["chain_probes"][f"{k}_{stop}"]


def test_frozen_chains():
    # reference test_generator.py:43-45
    crc = O.OParams(n=10, d=1)
    simple = O.OParams(n=10, d=1, kind=O.KIND_SIMPLE)
    v, pr = O.resolve_chain_block(simple, np.array([11], dtype=np.uint64), 0)
    assert (int(v[0]), pr) == (4, 2)
    v, pr = O.resolve_chain_block(crc, np.array([1001], dtype=np.uint64), 0)
    assert (int(v[0]), pr) == (286, 1)


def test_golden_n10_d2_both_engines():
    for kind, want in ((O.KIND_SIMPLE, GOLDEN_SIMPLE_N10_D2), (O.KIND_CRC, GOLDEN_CRC_N10_D2)):
        p = O.OParams(n=10, d=2, kind=kind)
        got, _ = O.generate_block(p, 0, p.m)
        assert [tuple(map(int, r)) for r in got] == want
        e = O.bb_generate(p)
        assert [tuple(map(int, r)) for r in e.reshape(-1, 2)] == want
    # reference test_generator.py:206-207
    got, _ = O.generate_block(O.OParams(n=10, d=2, kind=O.KIND_SIMPLE), 7, 8)
    assert tuple(map(int, got[0])) == (3, 2)


def test_72_combos_digests(golden):
    _, meta = golden
    seeds = {"none": (), "triangle": tuple(TRIANGLE.tolist()), "ring10": tuple(RING10.tolist())}
    assert len(meta["combos"]) == 72
    for c in meta["combos"]:
        p = O.OParams(n=c["n"], d=c["d"], n0=c["n0"], seed_edges=seeds[c["seed"]],
                      kind=O.KIND_CRC if c["kind"] == "crc" else O.KIND_SIMPLE)
        got, probes = O.generate_block(p, p.m0, p.m)
        assert _sha(got) == c["sha256"], c
        assert probes == c["probes"], c
        # the sequential BB fill (oracle.py:101-106) is the same array
        assert np.array_equal(O.bb_generate(p)[2 * p.m0:].reshape(-1, 2), got)


def test_config1_golden(golden):
    arrays, meta = golden
    g = meta["config1"]
    p = O.OParams(n=g["n"], d=g["d"])
    got, probes = O.generate_block(p, 0, p.m)
    assert _sha(got) == g["sha256"] and probes == g["probes"]
    assert np.array_equal(got[:4096], arrays["config1_head"])
    counts = np.zeros(p.n, dtype=np.int64)
    O.count_block(counts, got)
    assert _sha(counts) == g["counts_sha256"]
    assert int(counts.sum()) == g["degree_sum"] == 2 * p.m


def test_sampled_ids(golden):
    arrays, meta = golden
    for name, s in meta["samples"].items():
        p = O.OParams(n=s["n"], d=s["d"])
        ids = arrays[f"sample_{name}_ids"]
        r0 = np.uint64(2) * ids + np.uint64(1)
        for k in range(0, ids.size, 97):
            v, pr = O.resolve_chain_block(p, r0[k:k + 1], 0)
            assert pr == int(arrays[f"sample_{name}_probes"][k])
        vals, _ = O.resolve_chain_block(p, r0, 0)
        assert np.array_equal((vals >> np.uint64(1)) // np.uint64(s["d"]), arrays[f"sample_{name}_tgt"])


def test_window_subranges(golden):
    arrays, meta = golden
    for w in meta["windows"]:
        p = O.OParams(n=w["n"], d=w["d"])
        counts, probes = O.degree_block(p, w["lo"], w["hi"], w["K"])
        assert probes == w["probes"] and _sha(counts) == w["sha256"], w["name"]
        nz = np.nonzero(counts)[0]
        assert np.array_equal(nz, arrays[f"win_{w['name']}_idx"])


def test_full_counts(golden):
    arrays, meta = golden
    for f in meta["full"]:
        seed = tuple(f["seed"]) if f["seed"] else ()
        p = O.OParams(n=f["n"], d=f["d"], n0=f["n0"], seed_edges=seed)
        blk, probes = O.generate_block(p, p.m0, p.m)
        counts = np.zeros(p.n, dtype=np.int64)
        O.count_block(counts, blk)
        O.count_block(counts, np.array(seed, dtype=np.uint64).reshape(-1, 2))  # analytics.py:51-52, 98
        assert _sha(counts) == f["sha256"] and probes == f["probes"]
        assert int(counts.sum()) == f["sum"] == 2 * p.m


def test_threaded_driver_equals_serial():
    p = O.OParams(n=5000, d=7, n0=3, seed_edges=tuple(TRIANGLE.tolist()))
    want, wp = O.generate_block(p, p.m0, p.m)
    got, gp = O.run_threaded(p, p.m0, p.m, O.MODE_STORE, threads=4, batch=333)
    assert np.array_equal(got, want) and gp == wp
    counts, cp = O.run_threaded(p, p.m0, p.m, O.MODE_WINDOW, K=100, threads=3, batch=1000)
    ref = np.zeros(100, dtype=np.int64)
    O.count_block(ref, want)
    assert np.array_equal(counts, ref) and cp == wp
