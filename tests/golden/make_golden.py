"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``parba`` from ``/root/reference/pkg/src`` (numba cache redirected
to /tmp so nothing is written into the reference tree) and records its
outputs on seeded inputs into ``tests/golden/golden.npz`` and
``tests/golden/golden.json``.  The fixtures are committed; the GPU box never
reads /root/reference.  Inputs are seeded synthetic values with the shapes of
BASELINE.json's configs (there is no dataset for this path).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT_DIR = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "parba_numba_cache"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import parba  # noqa: F401
    from parba import _kernels, analytics, generator, hashing, oracle

    return hashing, generator, _kernels, analytics, oracle


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# (kind, seed0, seed1, salt, multiplier) -- the families the tests exercise
CFGS = [
    ("crc", 0, 1, 0, 3141592653589793238),
    ("crc", 7, 9, 0, 3141592653589793238),
    ("crc", 0, 1, 3, 3141592653589793238),
    ("crc", 2**40 + 5, 2**33 + 1, 0, 3141592653589793238),  # seeds truncate to 32 bits
    ("simple", 0, 1, 0, 3141592653589793238),
    ("simple", 0, 1, 5, 3141592653589793238),
]

TRIANGLE = [0, 1, 1, 2, 2, 0]
RING10 = [x for i in range(10) for x in (i, (i + 1) % 10)]


def main() -> None:
    hashing, generator, kernels, analytics, oracle = _import_reference()
    H = hashing
    rng = np.random.default_rng(160207106)
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"generated_by": "tests/golden/make_golden.py", "reference": REF_SRC, "cfgs": CFGS}

    def cfg_of(c):
        kind, s0, s1, salt, mult = c
        return H.HashConfig(kind=H.HashKind(kind), seed0=s0, seed1=s1, attempt_salt=salt, multiplier=mult)

    # -- CRC32-C primitive (hashing.py:105-116)
    seeds = rng.integers(0, 2**32, size=256, dtype=np.uint64)
    words = rng.integers(0, 2**64 - 1, size=256, dtype=np.uint64, endpoint=True)
    arrays["crc_seeds"] = seeds
    arrays["crc_words"] = words
    arrays["crc_out"] = np.array([H.crc32c_u64(int(s), int(w)) for s, w in zip(seeds, words)], dtype=np.uint64)
    arrays["crc_table"] = np.array(H.CRC32C_TABLE, dtype=np.uint32)

    # -- hash families (hashing.py:119-138) over several magnitudes + edges
    special = [1, 2, 3, 7, 11, 1000, 10**6, 2**31 - 1, 2**31, 2**32 - 1, 2**32, 2**32 + 1,
               2**40 + 13, 2**52 - 1, 2**52, 2**53 + 1, 2**63, 2**64 - 1]
    rs = np.concatenate([
        np.array(special, dtype=np.uint64),
        rng.integers(1, 1 << 12, size=400, dtype=np.uint64),
        rng.integers(1, 1 << 32, size=600, dtype=np.uint64),
        rng.integers(1, 1 << 42, size=600, dtype=np.uint64),
        rng.integers(1, 1 << 59, size=600, dtype=np.uint64),
        rng.integers(1, 2**64 - 1, size=200, dtype=np.uint64, endpoint=True),
    ])
    arrays["hash_r"] = rs
    for k, c in enumerate(CFGS):
        cfg = cfg_of(c)
        arrays[f"hash_out_{k}"] = np.array([H.hash_value(int(r), cfg) for r in rs], dtype=np.uint64)

    # -- chains (_kernels.py:121-135), total probes per (cfg, stop)
    r0s = rng.integers(1, 2**50, size=2000, dtype=np.uint64)
    arrays["chain_r0"] = r0s
    meta["chain_probes"] = {}
    for k, c in enumerate(CFGS):
        cfg = cfg_of(c)
        for stop in (0, 6, 1000):
            vals, probes = kernels.resolve_chain_block(r0s, stop, cfg)
            arrays[f"chain_out_{k}_{stop}"] = vals
            meta["chain_probes"][f"{k}_{stop}"] = int(probes)

    # -- generate_block digests for the 72 acceptance combos
    #    (tests/test_acceptance.py:36-54 of the reference)
    combos = []
    for n in (10**2, 10**3, 10**4):
        for d in (1, 2, 8, 16):
            for kind in ("crc", "simple"):
                for seed, n0 in ((None, 0), (TRIANGLE, 3), (RING10, 10)):
                    p = generator.GenParams(n=n, d=d, n0=n0,
                                            seed_edges=None if seed is None else np.array(seed, dtype=np.uint64),
                                            hash=H.HashConfig(kind=H.HashKind(kind)))
                    got, probes = generator.generate_block(p.m0, p.m, p)
                    want = oracle.edge_list(oracle.bb_generate(p, engine="python"), p.m0)
                    assert got.tobytes() == np.ascontiguousarray(want).tobytes()
                    combos.append({"n": n, "d": d, "kind": kind, "n0": n0,
                                   "seed": "none" if seed is None else ("triangle" if n0 == 3 else "ring10"),
                                   "sha256": sha(got), "probes": int(probes)})
    meta["combos"] = combos

    # -- config 1 (BASELINE.json configs[0]): n=1e5, d=4, full array
    p1 = generator.GenParams(n=10**5, d=4)
    c1, pr1 = generator.generate_block(0, p1.m, p1)
    counts1 = np.zeros(p1.n, dtype=np.int64)
    analytics.count_block(counts1, c1)
    meta["config1"] = {"n": 10**5, "d": 4, "sha256": sha(c1), "probes": int(pr1),
                       "degree_sum": int(counts1.sum()), "degree_max": int(counts1.max()),
                       "deg0_4": [int(x) for x in counts1[:5]], "last_edge": [int(x) for x in c1[-1]],
                       "counts_sha256": sha(counts1)}
    arrays["config1_head"] = c1[:4096].copy()
    arrays["config1_counts"] = counts1.astype(np.uint32)

    # -- sampled edge IDs at the large configs (per-id probes kept)
    meta["samples"] = {}
    for name, n, d in (("c2", 10**8, 10), ("c3", 10**9, 100), ("c4", 10**8, 16), ("c5", 10**10, 100)):
        p = generator.GenParams(n=n, d=d)
        ids = np.sort(rng.integers(0, p.m, size=2048, dtype=np.uint64))
        ids[:4] = [0, 1, p.m - 2, p.m - 1]
        ids = np.sort(ids)
        terms = np.empty_like(ids)
        probes = np.empty(ids.size, dtype=np.uint32)
        for k, i in enumerate(ids):
            v, pr = kernels.resolve_chain_block(np.array([2 * int(i) + 1], dtype=np.uint64), 0, p.hash)
            terms[k] = v[0]
            probes[k] = pr
            e = generator.generate_edge(int(i), p)
            assert e.target == (int(v[0]) >> 1) // d
        arrays[f"sample_{name}_ids"] = ids
        arrays[f"sample_{name}_src"] = ids // np.uint64(d)
        arrays[f"sample_{name}_tgt"] = (terms >> np.uint64(1)) // np.uint64(d)
        arrays[f"sample_{name}_probes"] = probes
        meta["samples"][name] = {"n": n, "d": d}

    # -- window histograms on subranges (generate_block + count_block)
    meta["windows"] = []
    for name, n, d, lo, hi, K in (
        ("c3_head", 10**9, 100, 0, 300_000, 10**5),
        ("c3_tail", 10**9, 100, 10**11 - 300_000, 10**11, 10**5),
        ("c5_tail", 10**10, 100, 10**12 - 200_000, 10**12, 10**5),
        ("c3_mid", 10**9, 100, 5 * 10**10, 5 * 10**10 + 200_000, 10**5),
    ):
        p = generator.GenParams(n=n, d=d)
        counts = np.zeros(K, dtype=np.int64)
        blk, probes = generator.generate_block(lo, hi, p)
        analytics.count_block(counts, blk)
        nz = np.nonzero(counts)[0]
        arrays[f"win_{name}_idx"] = nz.astype(np.uint32)
        arrays[f"win_{name}_val"] = counts[nz].astype(np.uint32)
        meta["windows"].append({"name": name, "n": n, "d": d, "lo": lo, "hi": hi, "K": K,
                                "probes": int(probes), "sum": int(counts.sum()),
                                "sha256": sha(counts)})

    # -- full degree counts (config-4 shape at desk scale), seed graph folded
    meta["full"] = []
    for n, d, seed, n0 in ((10**5, 16, None, 0), (2000, 3, TRIANGLE, 3), (3000, 5, RING10, 10)):
        p = generator.GenParams(n=n, d=d, n0=n0, seed_edges=None if seed is None else np.array(seed, dtype=np.uint64))
        counter, stats = analytics.degree_counts(p)
        meta["full"].append({"n": n, "d": d, "n0": n0, "seed": seed, "sha256": sha(counter.counts),
                             "sum": int(counter.counts.sum()), "probes": int(stats.hash_probes)})
        arrays[f"full_{n}_{d}_counts"] = counter.counts.astype(np.uint32)

    np.savez_compressed(os.path.join(OUT_DIR, "golden.npz"), **arrays)
    with open(os.path.join(OUT_DIR, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", OUT_DIR, "arrays:", len(arrays))


if __name__ == "__main__":
    main()
