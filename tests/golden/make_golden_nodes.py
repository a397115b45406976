"""Golden fixtures for the node-granular rows (f3 option flags,
f4 degree sequences), made by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_nodes.py

Like make_golden.py it imports ``parba`` from /root/reference/pkg/src with
the numba cache redirected to /tmp, and writes ``golden_nodes.npz`` /
``golden_nodes.json`` next to this file.  Every case is a seeded synthetic
family (degree sequences drawn from a seeded generator, seed graphs from the
reference's own test helpers' shapes).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import OUT_DIR, RING10, TRIANGLE, _import_reference, sha  # noqa: E402


def complete_edges(k: int) -> list[int]:
    return [x for u in range(k) for v in range(u + 1, k) for x in (u, v)]


def random_seed_graph(rng, k: int, m: int) -> list[int]:
    flat = [x for i in range(k) for x in (i, (i + 1) % k)]
    for _ in range(m):
        flat += [int(rng.integers(k)), int(rng.integers(k))]
    return flat


def main() -> None:
    hashing, generator, kernels, analytics, oracle = _import_reference()
    from parba import degreeseq, driver, errors

    H = hashing
    rng = np.random.default_rng(1602071060)
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"generated_by": "tests/golden/make_golden_nodes.py", "degseq": [], "flags": [],
                  "infeasible": [], "index": [], "counts": []}

    def hcfg(kind="crc", s0=0, s1=1, salt=0):
        return H.HashConfig(kind=H.HashKind(kind), seed0=s0, seed1=s1, attempt_salt=salt)

    # -- f4: generate_block with degree sequences (zeros included), three
    #    seed shapes, both hash kinds; all three resolutions must agree
    k = 0
    for n_nodes, max_deg, zero_frac in ((50, 4, 0.3), (700, 6, 0.2), (3000, 9, 0.1), (20000, 30, 0.05)):
        for kind in ("crc", "simple"):
            for seed, n0 in ((None, 0), (TRIANGLE, 3), (RING10, 10)):
                deg = rng.integers(1, max_deg + 1, size=n_nodes)
                deg[rng.random(n_nodes) < zero_frac] = 0
                deg[0] = max(int(deg[0]), 1)
                deg = deg.astype(np.uint64)
                p = generator.GenParams(n=n0 + n_nodes, n0=n0, degrees=deg,
                                        seed_edges=None if seed is None else np.array(seed, dtype=np.uint64),
                                        hash=hcfg(kind))
                blk, probes = generator.generate_block(p.m0, p.m, p)
                for res in ("bisect", "deferred"):
                    b2, p2 = generator.generate_block(p.m0, p.m, p, resolution=res)
                    assert np.array_equal(blk, b2) and p2 == probes
                name = f"deg{k}"
                arrays[f"{name}_degrees"] = deg
                if blk.shape[0] <= 40000:
                    arrays[f"{name}_edges"] = blk
                # an unaligned interior block too (plain mode is edge-granular)
                lo = p.m0 + (p.m - p.m0) // 3 + 1
                hi = lo + min(777, p.m - lo)
                sub, sp = generator.generate_block(lo, hi, p)
                meta["degseq"].append({"name": name, "kind": kind, "n0": n0,
                                       "seed": None if seed is None else list(seed), "n": p.n, "m": p.m,
                                       "sha256": sha(blk), "probes": int(probes),
                                       "sub": [lo, hi, sha(sub), int(sp)]})
                k += 1

    # -- f4: degree counts (window and full) with a degree sequence
    for name in ("deg3", "deg14"):
        c = next(x for x in meta["degseq"] if x["name"] == name)
        p = generator.GenParams(n=c["n"], n0=c["n0"], degrees=arrays[f"{name}_degrees"],
                                seed_edges=None if c["seed"] is None else np.array(c["seed"], dtype=np.uint64),
                                hash=hcfg(c["kind"]))
        for K in (None, max(1, p.n // 7)):
            counter, stats = analytics.degree_counts(p, K=K) if K else analytics.degree_counts(p)
            meta["counts"].append({"case": name, "K": K, "sha256": sha(counter.counts),
                                   "sum": int(counter.counts.sum()), "probes": int(stats.hash_probes)})

    # -- f4: the index itself (W, rank words, rank1, lookups)
    deg = rng.integers(0, 6, size=1500).astype(np.uint64)
    deg[0] = 3
    pi = degreeseq.build_prefix(deg, m0=5, n0=4)
    rb = degreeseq.build_rank_bits(pi)
    es = rng.integers(0, pi.m, size=3000, dtype=np.uint64)
    gen_es = rng.integers(pi.m0, pi.m, size=3000, dtype=np.uint64)
    arrays["index_degrees"] = deg
    arrays["index_W"] = pi.W
    arrays["index_words"] = rb.words
    arrays["index_es"] = es
    arrays["index_rank1"] = degreeseq.rank1_many(rb, es).astype(np.uint64)
    arrays["index_gen_es"] = gen_es
    arrays["index_owner"] = degreeseq.node_of_edge_many(gen_es, rb).astype(np.uint64)
    assert np.array_equal(arrays["index_owner"], degreeseq.node_of_edge_bisect_many(gen_es, pi))
    assert np.array_equal(arrays["index_owner"], degreeseq.owners_of_edges_deferred(gen_es, pi))
    meta["index"] = {"m0": 5, "n0": 4, "m": pi.m, "n_ones": rb.n_ones,
                     "owners": None if rb.owners is None else [int(x) for x in rb.owners[:8]]}

    # -- f3: option flags, uniform d and degree sequences, salted families
    f = 0
    cases = []
    for kind in ("crc", "simple"):
        for salt in (0, 5):
            cases.append(dict(n=200, d=3, n0=3, seed=TRIANGLE, nsl=True, npe=False, kind=kind, salt=salt))
            cases.append(dict(n=200, d=3, n0=4, seed=complete_edges(4), nsl=False, npe=True, kind=kind, salt=salt))
            cases.append(dict(n=150, d=2, n0=4, seed=complete_edges(4), nsl=True, npe=True, kind=kind, salt=salt))
    cases.append(dict(n=60, d=5, n0=6, seed=complete_edges(6), nsl=False, npe=True, kind="crc", salt=0))
    cases.append(dict(n=8, degrees=[3, 2, 4, 3, 1], n0=3, seed=TRIANGLE, nsl=False, npe=True, kind="crc", salt=0))
    for _ in range(3):
        kk = int(rng.integers(3, 12))
        seed = random_seed_graph(rng, kk, int(rng.integers(0, 8)))
        cases.append(dict(n=10**4, d=3, n0=kk, seed=seed, nsl=True, npe=False, kind="crc", salt=0))
        cases.append(dict(n=10**4, d=3, n0=kk, seed=seed, nsl=False, npe=True, kind="crc", salt=0))
    dg = rng.integers(0, 7, size=3000).astype(np.uint64)
    dg[0] = 2
    cases.append(dict(n=3005, degrees=dg.tolist(), n0=5, seed=complete_edges(5), nsl=True, npe=True, kind="crc",
                      salt=0))
    cases.append(dict(n=3005, degrees=dg.tolist(), n0=5, seed=complete_edges(5), nsl=True, npe=False,
                      kind="simple", salt=0))
    for c in cases:
        kw = dict(n=c["n"], n0=c["n0"], seed_edges=np.array(c["seed"], dtype=np.uint64),
                  no_self_loops=c["nsl"], no_parallel_edges=c["npe"], hash=hcfg(c["kind"], salt=c["salt"]))
        if "degrees" in c:
            kw["degrees"] = np.array(c["degrees"], dtype=np.uint64)
        else:
            kw["d"] = c["d"]
        p = generator.GenParams(**kw)
        blk, probes = generator.generate_block(p.m0, p.m, p)
        name = f"flag{f}"
        if blk.shape[0] <= 40000:
            arrays[f"{name}_edges"] = blk
        if "degrees" in c:
            arrays[f"{name}_degrees"] = kw["degrees"]
        entry = {k2: v for k2, v in c.items() if k2 != "degrees"}
        entry.update({"name": name, "m": p.m, "sha256": sha(blk), "probes": int(probes),
                      "has_degrees": "degrees" in c})
        # a node-aligned interior block
        v_lo = p.n0 + (p.n - p.n0) // 3
        v_hi = min(p.n, v_lo + 7)
        lo, hi = p.first_edge_of(v_lo), (p.m if v_hi == p.n else p.first_edge_of(v_hi))
        sub, sp = generator.generate_block(lo, hi, p)
        entry["sub"] = [lo, hi, sha(sub), int(sp)]
        # degree counts through the driver (node batches)
        counter, stats = analytics.degree_counts(p)
        entry["counts_sha256"] = sha(counter.counts)
        entry["counts_probes"] = int(stats.hash_probes)
        meta["flags"].append(entry)
        f += 1

    # -- f3: infeasible pools (InfeasibleTargetsError messages)
    for kw in (dict(n=3, d=3, n0=2, seed=[0, 1], max_attempts=None),
               dict(n=3, d=3, n0=2, seed=[0, 1], max_attempts=5)):
        p = generator.GenParams(n=kw["n"], d=kw["d"], n0=kw["n0"], seed_edges=np.array(kw["seed"], dtype=np.uint64),
                                no_self_loops=True, no_parallel_edges=True, max_attempts=kw["max_attempts"])
        try:
            generator.generate_block(p.m0, p.m, p)
            msg = None
        except errors.InfeasibleTargetsError as e:
            msg = str(e)
        meta["infeasible"].append({**kw, "message": msg})

    np.savez_compressed(os.path.join(OUT_DIR, "golden_nodes.npz"), **arrays)
    with open(os.path.join(OUT_DIR, "golden_nodes.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote golden_nodes: arrays", len(arrays), "degseq", len(meta["degseq"]), "flags", len(meta["flags"]))


if __name__ == "__main__":
    main()
