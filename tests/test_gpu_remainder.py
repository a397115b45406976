"""Exact h % r pinned directly (reference: _kernels.py:32-42, hashing.py:
119-125 -- the reference computes h % r exactly for every r).

Every tile kernel takes its remainder from one of the FP64-pipe routines of
parba_device.cuh (mod_fp31 / mod_fp<u32> / mod_fp<u64>, each with 1/r from
recip_approx or from phase 1's per-tile reciprocal series) or from mod_int.
These tests call those routines through parba_debug_mod(_check) on

* >= 1e8 device-drawn (h, r) pairs per routine and width class, including
  the paper's petaedge range r in [2^44, 2^52) (m = 1e15
  puts chain values near 2^50.8), against exact u64 %;
* an adversarial list (r in {1, 2, 3, 2^k +- 1, 2^31 - 1, 2^32 +- 1, 2^44,
  2^52 - 1}, h in {q*r - 1, q*r, q*r + 1}, halves 0xFFFFFFFF) against
  Python's exact integers;

and then run the tile kernels themselves at the paper's scale (n = 1e13,
d = 100: 2m ~ 2^50.8, the 5-chunk kernel) and at 2m just below 2^52,
store and window subranges vs the oracle.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_1602_07106_b200")
L_ = pb._lib

RY_MIN = (1 << 27) + 224  # the series path runs for tiles with 2*base >= 2^27
ONESTAGE_MIN = (1 << 28) + 224  # 2-chunk tiles with 2*base >= 2^28: one-stage remainder

# (method, rmin, rmax): each routine over the r range of the launches that use it
CLASSES = [
    (L_.MOD_FP31, 1, (1 << 31) - 1),
    (L_.MOD_FP_NARROW, 1, (1 << 32) - 1),
    (L_.MOD_FP_WIDE, 1, (1 << 52) - 1),
    (L_.MOD_FP_WIDE, 1 << 44, (1 << 52) - 1),  # petaedge chain values
    (L_.MOD_INT, 1, (1 << 64) - 1),
    (L_.MOD_FP31_SERIES, RY_MIN, (1 << 31) - 1),
    (L_.MOD_FP_NARROW_SERIES, RY_MIN, (1 << 32) - 1),
    (L_.MOD_FP_WIDE_SERIES, RY_MIN, (1 << 52) - 1),
    (L_.MOD_FP_WIDE_SERIES, 1 << 44, (1 << 52) - 1),
    (L_.MOD_FP31_SERIES1, ONESTAGE_MIN, (1 << 31) - 1),
    (L_.MOD_FP_WIDE_SERIES1, ONESTAGE_MIN, (1 << 52) - 1),
    (L_.MOD_FP_WIDE_SERIES1, 1 << 44, (1 << 52) - 1),
    (L_.MOD_FP32, 1, 0xF0000000),            # 3-chunk launches: the 32-bit tail
    (L_.MOD_FP32, 0xE0000000, 0xF0000000),   # at the top of its range, |t| closest to 2^31
    (L_.MOD_FP32_SERIES, RY_MIN, 0xF0000000),
    (L_.MOD_FP32_SERIES, 0xE0000000, 0xF0000000),
]


@pytest.mark.parametrize("method,rmin,rmax", CLASSES)
def test_remainder_random_1e8(method, rmin, rmax):
    import torch

    dev = torch.device("cuda", 0)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    first = torch.zeros(3, dtype=torch.int64, device=dev)
    total = 0
    for seed in (1, 2):  # 2 x 6e7 = 1.2e8 pairs per class
        pb._lib.check(pb._lib.load().parba_debug_mod_check(method, seed * 0x9E3779B9 + method, 60_000_000, rmin,
                                                           rmax, bad.data_ptr(), first.data_ptr(),
                                                           pb._lib.stream_ptr(torch, dev)))
        total += 60_000_000
    torch.cuda.synchronize()
    h, r, got = (int(x) & ((1 << 64) - 1) for x in first.cpu().tolist())
    assert int(bad.item()) == 0, f"{int(bad.item())} of {total} wrong, e.g. {h} % {r} = {h % r}, got {got}"


def _adversarial(rmin: int, rmax: int):
    rs = {1, 2, 3, (1 << 31) - 1, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, 1 << 44, (1 << 52) - 1,
          (1 << 63) + 1, (1 << 64) - 1, RY_MIN, RY_MIN + 1, ONESTAGE_MIN, ONESTAGE_MIN + 1}
    for k in range(1, 64):
        rs |= {(1 << k) - 1, 1 << k, (1 << k) + 1}
    rng = np.random.default_rng(160207106)
    rs |= {int(x) for x in rng.integers(1, 1 << 62, 64)}
    rs |= {rmin + int(x) % (rmax - rmin + 1) for x in rng.integers(0, 1 << 62, 16)}  # inside every class
    rs = sorted(r for r in rs if rmin <= r <= rmax)
    hs, rr = [], []
    M = (1 << 64) - 1
    for r in rs:
        cands = {0, 1, M, 0xFFFFFFFF, 0xFFFFFFFF00000000, 0xFFFFFFFF0000FFFF, r - 1, r, r + 1, 2 * r - 1}
        for q in (1, 2, 3, (1 << 32) - 1, 1 << 32, M // r, (M // r) // 2 + 1, int(rng.integers(1, 1 << 62))):
            cands |= {q * r - 1, q * r, q * r + 1}
        for h in cands:
            if 0 <= h <= M:
                hs.append(h)
                rr.append(r)
    return np.array(hs, dtype=np.uint64), np.array(rr, dtype=np.uint64)


@pytest.mark.parametrize("method,rmin,rmax", CLASSES)
def test_remainder_adversarial(method, rmin, rmax):
    import torch

    dev = torch.device("cuda", 0)
    h, r = _adversarial(rmin, rmax)
    hhi = torch.from_numpy((h >> np.uint64(32)).astype(np.uint32).view(np.int32)).to(dev)
    hlo = torch.from_numpy((h & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)).to(dev)
    rd = torch.from_numpy(r.view(np.int64)).to(dev)
    out = torch.empty(h.size, dtype=torch.int64, device=dev)
    pb._lib.check(pb._lib.load().parba_debug_mod(method, hhi.data_ptr(), hlo.data_ptr(), rd.data_ptr(), h.size,
                                                 out.data_ptr(), pb._lib.stream_ptr(torch, dev)))
    got = out.cpu().numpy().view(np.uint64)
    want = h % r  # numpy uint64 % is exact integer division
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(int(h[k]), int(r[k]), int(got[k]), int(want[k])) for k in bad[:5]]
    assert h.size > 200


def test_rcp_approx_bound_exhaustive():
    """rcp.approx.ftz.f64 reads only the high word of its operand, so its
    relative error over every operand in [1, 2^64) is the maximum over 2^20
    mantissa prefixes x 64 exponents x both ends of the low word.  The
    remainder analysis (parba_device.cuh: mod_fp_y, mod_fp31_y1) assumes
    < 2^-19.5 raw and < 2^-38 after the Newton step."""
    import torch

    dev = torch.device("cuda", 0)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    pb._lib.check(pb._lib.load().parba_debug_rcp_bound(1023, 64, out.data_ptr(), pb._lib.stream_ptr(torch, dev)))
    raw, newton = out.cpu().tolist()
    assert 0 < raw < 2.0 ** -19.5, raw
    assert newton < 2.0 ** -38, newton


def _op(p):
    return O.OParams(n=p.n, d=p.d, n0=p.n0, seed_edges=tuple(int(x) for x in p.seed_edges))


# the paper's petaedge graph (m = 1e15) and 2m just below 2^52
PETA = [(10**13, 100), (((1 << 51) - 1) // 1000, 1000)]


@pytest.mark.parametrize("n,d", PETA)
def test_store_subranges_at_petaedge_scale(n, d):
    """Tile-kernel store mode (5-chunk CRC, mod_fp<u64> and the series) on
    ragged subranges at the top, middle and 2^32 boundary region of the ID
    space vs the oracle."""
    import torch

    p = pb.GenParams(n=n, d=d)
    assert (1 << 44) < 2 * p.m < (1 << 52)
    dev = torch.device("cuda", 0)
    for lo, hi in ((p.m - 1_000_003, p.m), (p.m // 2 + 17, p.m // 2 + 700_000), ((1 << 31) - 5000, (1 << 31) + 300_001),
                   ((1 << 43) + 11, (1 << 43) + 500_000)):
        got, prb = pb.generate_block_device(lo, hi, p, device=dev)
        want, wp = O.generate_block(_op(p), lo, hi)
        assert np.array_equal(got.cpu().numpy().view(np.uint64), want), (lo, hi)
        assert int(prb.item()) == wp
        host, hp = pb.generate_block(lo, hi, p)  # the host-array pipeline, same launch widths
        assert np.array_equal(host, want) and hp == wp


@pytest.mark.parametrize("n,d", PETA)
def test_window_subranges_at_petaedge_scale(n, d):
    """The streaming window (K = 1e5, the paper's demo) on top-of-range and
    low subranges of the petaedge graph vs the oracle, counts and probes."""
    p = pb.GenParams(n=n, d=d)
    K = 10**5
    for lo, hi in ((p.m - 2_000_000, p.m), (0, 3_000_000), (p.m // 3, p.m // 3 + 1_000_000)):
        counts, probes = pb.parallel.count_shard_device(p, K, lo, hi)
        want, wp = O.degree_block(_op(p), lo, hi, K)
        assert np.array_equal(counts.cpu().numpy(), want), (lo, hi)
        assert int(probes.item()) == wp


def test_sampled_ids_at_petaedge_scale():
    p = pb.GenParams(n=10**13, d=100)
    ids = np.random.default_rng(160207106).integers(0, p.m, 200_000, dtype=np.uint64)
    got, pr = pb.edges_at(ids, p)
    r, wp = O.resolve_chain_block(_op(p), 2 * ids + np.uint64(1), 0)
    assert np.array_equal(got[:, 1], (r >> np.uint64(1)) // np.uint64(p.d))
    assert np.array_equal(got[:, 0], ids // np.uint64(p.d)) and pr == wp
