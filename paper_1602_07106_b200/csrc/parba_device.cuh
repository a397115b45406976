// parba_device.cuh -- device-side building blocks of the B200 hot path.
//
//   crc_chunks    CRC32-C of one 64-bit word with seed s0 from 11-bit chunk
//                 tables in shared memory: 3 lookups for positions < 2^32, 4
//                 for < 2^43; offsets by shift+mask on the ALU pipe.
//   crc_bytes     byte-sliced variant for the generic kernels (any 64-bit value).
//   h_crc(r)      the reference hash ((crc(s0,r)<<32) + crc(s1,r)) % r
//                 (hashing.py:119-125, _kernels.py:32-42) rewritten through
//                 CRC linearity: crc(s,w) = crc(s,0) ^ crc(0,w), so one table
//                 CRC per probe instead of the reference's two.
//   mod_fp(h,r)   exact h % r for r < 2^52, computed on the FP64 pipe (64
//                 lanes/SM/clk on B200, otherwise idle), which keeps the ALU
//                 and FMA pipes free for the CRC and the chain bookkeeping.
//   mod_int(h,r)  exact h % r for any 64-bit r (generic kernels).
//   h_simple(r)   umulhi((r*M) mod 2^64, r)  (hashing.py:128-138).
//   Magic32/64    division by the launch-constant d (closed forms for
//                 source/target, generator.py:157-169) by multiply-high.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace parba {

// Debug builds (-DPARBA_DEBUG_CHECKS=1, tools/check_build.sh) trap on a
// violated invariant; release builds compile the checks away.
#if defined(PARBA_DEBUG_CHECKS) && PARBA_DEBUG_CHECKS
#define PARBA_CHECK(cond)                \
    do {                                 \
        if (!(cond)) __trap();           \
    } while (0)
#else
#define PARBA_CHECK(cond) \
    do {                  \
    } while (0)
#endif

constexpr uint32_t kCrcPoly = 0x82F63B78u;  // hashing.py:40 (reflected 0x1EDC6F41)

// Bit-serial CRC32-C of one LE 64-bit word (host + device); builds tables
// and the seed constants only.
__host__ __device__ inline uint32_t crc32c_u64_bitwise(uint32_t seed, uint64_t word) {
    uint32_t c = seed;
    for (int b = 0; b < 64; ++b) {
        uint32_t bit = (c ^ (uint32_t)(word >> b)) & 1u;
        c = (c >> 1) ^ (kCrcPoly & (0u - bit));
    }
    return c;
}

// ---------------------------------------------------------------------------
// Division by a runtime-invariant d >= 1.
//   Magic64: Granlund-Montgomery round-up form for any 64-bit n:
//            t = mulhi(mul, n);  q = (t + ((n - t) >> sh1)) >> sh2
//   Magic32: n < 2^31 (every narrow position), d < 2^31: with
//            l = ceil(log2 d), m = floor(2^(31+l)/d) + 1 < 2^32,
//            q = (n*m) >> (31+l) exactly (Granlund-Montgomery, N = 31):
//            one IMAD.WIDE.U32 and one funnel shift.
struct Magic64 {
    uint64_t mul;
    uint32_t sh1, sh2;
};
struct Magic32 {
    uint32_t mul, shift;
};

inline Magic64 make_magic64(uint64_t d) {
    Magic64 m{};
    int l = 0;
    while (l < 64 && (1ull << l) < d) ++l;  // l = ceil(log2 d)
    unsigned __int128 num = ((unsigned __int128)1 << 64) * (((unsigned __int128)1 << l) - d);
    m.mul = (uint64_t)(num / d) + 1;
    m.sh1 = l > 0 ? 1u : 0u;
    m.sh2 = l > 0 ? (uint32_t)(l - 1) : 0u;
    return m;
}

inline Magic32 make_magic32(uint64_t d) {
    Magic32 m{};
    if (d < 1 || d >= (1ull << 31)) return m;  // narrow launches need d < 2^31
    int l = 0;
    while ((1ull << l) < d) ++l;
    m.mul = (uint32_t)((1ull << (31 + l)) / d + 1);
    m.shift = (uint32_t)(31 + l);
    return m;
}

__device__ __forceinline__ uint64_t magic_div(uint64_t n, const Magic64 &m) {
    uint64_t t = __umul64hi(m.mul, n);
    return (t + ((n - t) >> m.sh1)) >> m.sh2;
}
// n < 2^31
__device__ __forceinline__ uint32_t magic_div32(uint32_t n, const Magic32 &m) {
    return (uint32_t)(((uint64_t)n * m.mul) >> m.shift);
}

// Launch-constant description of one graph family (plain uniform-d mode).
struct DevParams {
    uint64_t n, d, n0, m0, m;
    uint64_t stop;         // 2*m0: chains stop when r < stop (seed region)
    uint64_t mult;         // SIMPLE multiplier
    uint32_t k0, k01;      // crc(s0,0) and crc(s0,0)^crc(s1,0): h = (c0<<32)|(c0^k01)
    const uint64_t *seed;  // 2*m0 seed endpoints (device)
    Magic64 div64;         // by d (wide)
    Magic32 div32;         // by d (narrow: positions < 2^31)
    Magic32 div32_2d;      // by 2d (every r < 2^31: target = (r - 2m0) / 2d + n0)
    uint64_t win_rlim;     // window mode: generated target < K  <=>  r < win_rlim
    uint32_t win_rlim32;   // min(win_rlim, 2^32 - 1) for narrow launches
    uint32_t tgt_fp;       // wide launches: targets by the FP64 reciprocal (target_fp)
    uint32_t win_fp;       // window hits (targets < K <= 2^32) by target_fp
    double inv2d;          // RN(1 / (2d))
    uint64_t K;
    // degree sequences (f4): node of a position by rank (degreeseq.py:145-178)
    const uint64_t *W;         // W[k] = first edge of node n0+k, W[n-n0] = m
    const ulonglong2 *rank;    // per 64 positions: {start bits, ones before}
    const uint64_t *owners;    // rank -> node, NULL when every degree >= 1
    const uint32_t *dense;     // optional: owning node of every generated position (m - m0 entries, n < 2^32)
};

// Rank directory of a degree sequence: one 16-byte entry per 64 positions,
// x = bit j set iff a node with degree >= 1 starts at position 64w+j,
// y = number of such starts before position 64w.  One LDG.128 per lookup
// (the reference's two-level 512-bit superblock directory, degreeseq.py:
// 118-151, traded for a single sector read).
__device__ __forceinline__ uint64_t rank1_dev(const ulonglong2 *rank, uint64_t e) {
    const ulonglong2 w = __ldg(rank + (e >> 6));
    const uint64_t mask = ~(0xFFFFFFFFFFFFFFFEull << (e & 63));  // bits 0..e&63
    return w.y + (uint64_t)__popcll(w.x & mask);
}
// Random 4-byte read of the dense owner map.  PARBA_DENSE_LD selects the
// load form (0: ld.global.nc; 1: no L1 allocation + 64-byte L2 fetch hint).
#ifndef PARBA_DENSE_LD
#define PARBA_DENSE_LD 1
#endif
__device__ __forceinline__ uint32_t ld_dense(const uint32_t *ptr) {
#if PARBA_DENSE_LD == 1
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(ptr));
    return v;
#else
    return __ldg(ptr);
#endif
}

// Owning node of generated position e (m0 <= e < m): node_of_edge
// (degreeseq.py:165-178) -- the last node with W <= e and degree >= 1.
// With the dense map (4 bytes per position, parba_degseq_dense) a lookup is
// one independent 4-byte load instead of a rank entry and an owners gather.
__device__ __forceinline__ uint64_t node_of(uint64_t e, const DevParams &p) {
    if (p.dense) return ld_dense(p.dense + (e - p.m0));
    const uint64_t r = rank1_dev(p.rank, e);
    return p.owners ? __ldg(p.owners + r - 1) : p.n0 + r - 1;
}

// Closed forms (generator.py:157-169): source of edge i, target of terminal r.
// DEG: degree sequence, node_of instead of the division by d.
template <bool NARROW, bool SEED, bool DEG = false>
__device__ __forceinline__ uint64_t source_of(uint64_t i, const DevParams &p) {
    if constexpr (DEG) return node_of(i, p);
    if constexpr (NARROW) {
        if constexpr (SEED) return (uint64_t)magic_div32((uint32_t)(i - p.m0), p.div32) + p.n0;
        else return (uint64_t)magic_div32((uint32_t)i, p.div32);
    } else {
        if constexpr (SEED) return magic_div(i - p.m0, p.div64) + p.n0;
        else return magic_div(i, p.div64);
    }
}
// R31: every chain value < 2^31, so floor(((r>>1) - m0)/d) = floor((r - 2m0)/(2d))
// is one 32-bit multiply-high division.
template <bool NARROW, bool SEED, bool R31 = false, bool DEG = false>
__device__ __forceinline__ uint64_t target_of(uint64_t r, const DevParams &p) {
    if constexpr (SEED) {
        if (r < p.stop) return __ldg(p.seed + r);
    }
    if constexpr (DEG) return node_of(r >> 1, p);
    if constexpr (R31) {
        if constexpr (SEED) return (uint64_t)magic_div32((uint32_t)(r - p.stop), p.div32_2d) + p.n0;
        else return (uint64_t)magic_div32((uint32_t)r, p.div32_2d);
    }
    return source_of<NARROW, SEED>(r >> 1, p);
}

// Target of a terminal value r < 2^52 (wide launches) without a 64-bit
// integer division: q = floor((r - 2m0) / 2d) + n0 (generator.py:163-169) as
// round(x * RN(1/2d) - 1/2 + 2^-19) with x = r - 2m0 exact in a double (the
// rounding by the 1.5*2^52 magic addition).  For
// q < 2^32 the product and the first rounding err by at most 2^-20, so the
// value lies in [Q + phi - 1/2 + 2^-20, Q + phi - 1/2 + 3*2^-20] (phi = the
// fraction, 0 <= phi <= 1 - 1/2d) and rounds to Q whenever 3*2^-20 < 1/2d,
// i.e. d < 174762 (the host checks that and n <= 2^32: DevParams.tgt_fp).
template <bool SEED>
__device__ __forceinline__ uint64_t target_fp(uint64_t r, const DevParams &p) {
    if constexpr (SEED) {
        if (r < p.stop) return __ldg(p.seed + r);
        r -= p.stop;
    }
    const double x = __longlong_as_double((long long)(r | 0x4330000000000000ull)) - 0x1p52;  // exact, r < 2^52
    // + 1.5*2^52 keeps every sum (>= -1/2) in [2^52, 2^53), where the spacing
    // is 1: the addition rounds to the integer floor(x / 2d) in the low word
    const double q = fma(x, p.inv2d, -0.5 + 0x1p-19) + 0x1.8p52;
    const uint64_t t = (uint64_t)(uint32_t)__double2loint(q);  // floor(x / 2d) < 2^32
    if constexpr (SEED) return t + p.n0;
    else return t;
}

// ---------------------------------------------------------------------------
// Exact remainder.

// Exact integer -> double: I2F.F64 (one XU instruction) or the magic-exponent
// trick (MOV + DADD on the FP64 pipe).  The mix used by mod_fp31 is a tuning
// knob (PARBA_CVT31, bit k = operand k via magic: 1 r, 2 hhi, 4 hlo).
__device__ __forceinline__ double u32_to_f64_magic(uint32_t x) {
    return __hiloint2double(0x43300000, (int)x) - 0x1p52;
}
__device__ __forceinline__ double u32_to_f64_i2f(uint32_t x) { return __uint2double_rn(x); }
#ifndef PARBA_ROT
#define PARBA_ROT 0
#endif
#ifndef PARBA_CVT31
#define PARBA_CVT31 6
#endif
template <int BIT>
__device__ __forceinline__ double cvt31(uint32_t x) {
    if constexpr ((PARBA_CVT31 >> BIT) & 1) return u32_to_f64_magic(x);
    else return u32_to_f64_i2f(x);
}
__device__ __forceinline__ double u32_to_f64(uint32_t x) {
#ifdef PARBA_MAGIC_CVT
    return __hiloint2double(0x43300000, (int)x) - 0x1p52;
#else
    return __uint2double_rn(x);
#endif
}
#ifndef PARBA_CVTW
#define PARBA_CVTW 0
#endif
// chain value (< 2^52) of the wide kernels -> double; PARBA_CVTW bit 1: magic
__device__ __forceinline__ double r_to_f64w(uint64_t x) {
#if PARBA_CVTW & 2
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 0x1p52;
#else
    return __ull2double_rn(x);
#endif
}
__device__ __forceinline__ double u52_to_f64(uint64_t x) {  // x < 2^52
#ifdef PARBA_MAGIC_CVT
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 0x1p52;
#else
    return __ull2double_rn(x);
#endif
}

// hi:lo -> nearest double (one rounding).
__device__ __forceinline__ double u64_halves_to_f64(uint32_t hi, uint32_t lo) {
    double dh = __hiloint2double(0x45300000, (int)hi);  // 2^84 + hi*2^32
    double dl = __hiloint2double(0x43300000, (int)lo);  // 2^52 + lo
    return (dh - 0x1.00000001p84) + dl;                  // 2^84 + 2^52 exactly
}

// y ~ 1/rd: rcp.approx.ftz.f64 (max relative error 2^-19.9 measured on
// B200 by tools/micro) plus one Newton step: relative error < 2^-39.
__device__ __forceinline__ double recip_approx(double rd) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rd));
    const double e = fma(-rd, y, 1.0);
    return fma(y, e, y);
}

// h % r for 1 <= r < 2^52, h = hhi:hlo, entirely in fp64.
//   A: qa = round(hhi*y) is floor(hhi/r) or +1 (hhi/r < 2^32, error < 2^-7);
//      x = fma(-qa, r, hhi) is EXACT (the true value lies in [-r, r), which
//      a double holds exactly since r < 2^52) -- no correction needed yet.
//   B: v = x*2^32 + hlo (|v| < r*2^32); qb = round(v*y) is floor(v/r) or +1;
//      t = fma(-qb, r, x*2^32) + hlo is again exact, t in [-r, r);
//      one "if negative add r" gives h % r (= v % r, since v = h - qa*r*2^32).
// The 1.5*2^52 offset rounds q to an integer for |q| < 2^51 of either sign.
template <class R>
__device__ __forceinline__ R mod_fp_y(uint32_t hhi, uint32_t hlo, double rd, double y) {
    // the hash halves by the magic exponent (DADD) -- the XU pipe is the
    // busiest one in the wide kernels (I2F, MUFU, POPC); PARBA_CVTW bit 0:
    // halves via I2F instead
#if PARBA_CVTW & 1
    const double ha = u32_to_f64_i2f(hhi);
    const double hl = u32_to_f64_i2f(hlo);
#else
    const double ha = u32_to_f64_magic(hhi);
    const double hl = u32_to_f64_magic(hlo);
#endif
    const double qa = fma(ha, y, 0x1.8p52) - 0x1.8p52;
    const double x = fma(-qa, rd, ha);
    const double qb = fma(fma(x, 0x1p32, hl), y, 0x1.8p52) - 0x1.8p52;
    double t = fma(-qb, rd, x * 0x1p32) + hl;
    t = (t < 0.0) ? t + rd : t;
    const double tt = t + 0x1p52;  // t < 2^52: the mantissa holds t exactly
    const uint32_t lo = (uint32_t)__double2loint(tt);
    if constexpr (sizeof(R) == 4) {
        return lo;
    } else {
        const uint32_t hi = (uint32_t)__double2hiint(tt) & 0x000FFFFFu;
        return ((uint64_t)hi << 32) | lo;
    }
}
template <class R>
__device__ __forceinline__ R mod_fp(uint32_t hhi, uint32_t hlo, double rd) {
    return mod_fp_y<R>(hhi, hlo, rd, recip_approx(rd));
}

// h % r for 1 <= r < 2^31 (h = hhi:hlo): stage A as in mod_fp, then the
// final remainder in 32-bit integer arithmetic.  t = v - qb*r lies in [-r, r)
// and v = x*2^32 + hlo == hlo (mod 2^32), so t = hlo - qb*r (mod 2^32) read as
// int32 is exact (|t| < 2^31); t < 0 ? t + r : t == min_u32(t, t + r).  -qb is
// the low word of fma(-v, y, 1.5*2^52) (round-to-nearest is symmetric), so
// t = hlo + (-qb)*r needs no negation.
// 10 FP64 instructions + 1 IMAD + 2 ALU, no FP64 -> integer conversion.
__device__ __forceinline__ uint32_t mod_fp31_y(uint32_t hhi, uint32_t hlo, uint32_t r, double rd,
                                               double y) {
    const double ha = cvt31<1>(hhi);
    const double qa = fma(ha, y, 0x1.8p52) - 0x1.8p52;
    const double x = fma(-qa, rd, ha);                          // exact, in [-r, r)
    const double v = fma(x, 0x1p32, cvt31<2>(hlo));             // ~ x*2^32 + hlo
    const uint32_t nqb = (uint32_t)__double2loint(fma(-v, y, 0x1.8p52));  // -qb mod 2^32
    const uint32_t t = hlo + nqb * r;                           // exact mod 2^32
    return min(t, t + r);
}
// The same for 1 <= r <= kR32Max (3-chunk launches: chain values < 2^32).
// With y ~ 1/r to a relative error < 2^-37.6 (recip_approx: 2^-39; the tile
// series adds (224/2^27)^2) and v = RN(V), V = x*2^32 + hlo (|v - V| < r*2^-21):
// |v*y - V/r| < 2^32 * 2^-37.6 + 2^-21 < 0.0207, so qb = round(v*y) gives
// t = V - qb*r with |t| <= 0.5207 r < 2^31 for r <= kR32Max = 0.9375 * 2^32:
// t = hlo - qb*r (mod 2^32) read as int32 is exact, and t < 0 ? t + r : t is
// the remainder.  3 integer instructions instead of mod_fp's ~9 FP64 ones
// for the second stage (PARBA_R32=0: 3-chunk launches keep mod_fp, A/B).
#ifndef PARBA_R32
#define PARBA_R32 1
#endif
constexpr uint32_t kR32Max = 0xF0000000u;
__device__ __forceinline__ uint32_t mod_fp32_y(uint32_t hhi, uint32_t hlo, uint32_t r, double rd, double y) {
    const double ha = cvt31<1>(hhi);
    const double qa = fma(ha, y, 0x1.8p52) - 0x1.8p52;
    const double x = fma(-qa, rd, ha);                          // exact, in [-r, r)
    const double v = fma(x, 0x1p32, cvt31<2>(hlo));
    const uint32_t nqb = (uint32_t)__double2loint(fma(-v, y, 0x1.8p52));  // -qb mod 2^32
    const uint32_t t = hlo + nqb * r;                           // t mod 2^32, |t| < 2^31
    return t + (r & (uint32_t)((int32_t)t >> 31));
}
#ifndef PARBA_ONESTAGE
#define PARBA_ONESTAGE 1
#endif
// 4- and 5-chunk tiles too (A/B: C3 window -2.6%, the integer correction
// costs more than the FP64 stages it saves there; off)
#ifndef PARBA_ONESTAGE_WIDE
#define PARBA_ONESTAGE_WIDE 0
#endif
#ifndef PARBA_ONESTAGE_WIDE_STORE
#define PARBA_ONESTAGE_WIDE_STORE 1
#endif
constexpr uint64_t kOneStageMin = 1ull << 28;
// One-stage form for 2^28 <= r < 2^31 (phase 1 of 2-chunk tiles with 2*base
// >= kOneStageMin): q = round(v), v = hd*y, from h rounded to a double hd
// (|hd - h| <= 2^11, i.e. <= 2^-17 in v) and y ~ 1/r with relative error
// eps: |v - h/r| <= (h/r)*eps + 2^-17 with h/r < 2^36.  The tile series gives
// eps < 2^-38.6: Newton on an rcp.approx whose relative error is < 2^-19.5
// (2^-39 after the step; the raw bound is checked exhaustively over the
// instruction's 2^21 operands per exponent by parba_debug_rcp_bound) plus the
// series truncation (224/2^28)^2 = 2^-40.4.  So |v - h/r| < 0.17 < 1/2 and q
// is floor(h/r) or floor(h/r) + 1: t = hlo - q*r (mod 2^32) lies in [-r, r)
// and min(t, t + r) is the remainder, as in mod_fp31_y.  4 FP64 instructions
// instead of 7 (and no rd).
// PARBA_Y1_I2F: hd by one 64-bit I2F (XU pipe) instead of two magic-exponent
// conversions and an FMA (2 MOV + 2 DADD + DFMA): same single rounding (A/B)
#ifndef PARBA_Y1_I2F
#define PARBA_Y1_I2F 1
#endif
__device__ __forceinline__ double h_to_f64(uint32_t hhi, uint32_t hlo) {
#if PARBA_Y1_I2F
    return __ull2double_rn(((uint64_t)hhi << 32) | hlo);
#else
    return fma(u32_to_f64_magic(hhi), 0x1p32, u32_to_f64_magic(hlo));
#endif
}
__device__ __forceinline__ uint32_t mod_fp31_y1(uint32_t hhi, uint32_t hlo, uint32_t r, double y) {
    const double hd = h_to_f64(hhi, hlo);  // h, one rounding
    const uint32_t nq = (uint32_t)__double2loint(fma(-hd, y, 0x1.8p52));             // -q mod 2^32
    const uint32_t t = hlo + nq * r;
    return min(t, t + r);
}
// The one-stage form for 2^28 <= r < 2^52 (phase 1 of 3-chunk tiles with
// 2*base >= kOneStageMin; 4- and 5-chunk tiles with PARBA_ONESTAGE_WIDE): q = round(hd*y) as above (h/r < 2^36,
// |q - h/r| < 0.17 + 1/2), read whole from the mantissa of 2^52 + q, and t =
// h - q*r in 64-bit integer arithmetic (its true value lies in [-r, r), so
// the wrapping product is harmless); one correction.  4 FP64 instructions
// and ~8 integer ones instead of ~13 FP64 ones.
__device__ __forceinline__ uint64_t mod_fp_y1w(uint32_t hhi, uint32_t hlo, uint64_t r, double y) {
    const double hd = h_to_f64(hhi, hlo);
    const uint64_t q = (uint64_t)__double_as_longlong(fma(hd, y, 0x1p52)) - 0x4330000000000000ull;
    int64_t t = (int64_t)((((uint64_t)hhi << 32) | hlo) - q * r);
    t += (t < 0) ? (int64_t)r : 0;
    return (uint64_t)t;
}
__device__ __forceinline__ uint32_t mod_fp31(uint32_t hhi, uint32_t hlo, uint32_t r) {
    const double rd = cvt31<0>(r);
    return mod_fp31_y(hhi, hlo, r, rd, recip_approx(rd));
}

// h % r for any 1 <= r < 2^64 (generic kernels; integer corrections).
__device__ __forceinline__ uint64_t mod_int(uint32_t hhi, uint32_t hlo, uint64_t r) {
    const uint64_t h = ((uint64_t)hhi << 32) | hlo;
    if (r > (1ull << 63)) return h >= r ? h - r : h;   // h < 2^64 < 2r
    const double rd = u64_halves_to_f64((uint32_t)(r >> 32), (uint32_t)r);
    const double y = recip_approx(rd);
    const uint32_t qa = (uint32_t)__double2loint(fma(u32_to_f64(hhi), y, 0x1p52));
    int64_t x = (int64_t)((uint64_t)hhi - (uint64_t)qa * r);
    x += (x < 0) ? (int64_t)r : 0;                     // x = hhi mod r < 2^32
    const uint64_t v = ((uint64_t)x << 32) | hlo;      // < r * 2^32, no overflow
    // qb = round(v / r) may be 2^32 itself (x = r - 1, hlo near 2^32 - 1, r <=
    // 2^32): read all of it from the mantissa of 2^52 + qb, not its low word
    const uint64_t qb = (uint64_t)__double_as_longlong(fma(u64_halves_to_f64((uint32_t)x, hlo), y, 0x1p52)) -
                        0x4330000000000000ull;
    int64_t t = (int64_t)(v - qb * r);                 // in [-r, r) (mod 2^64 arithmetic), r <= 2^63
    t += (t < 0) ? (int64_t)r : 0;
    return (uint64_t)t;
}

// ---------------------------------------------------------------------------
// CRC tables in shared memory.  Table 0 of every layout carries
// k0 = crc(s0, 0): each crc() XORs exactly one table-0 entry, so it returns
// crc(s0, w) directly (CRC linearity).
//
// Byte layout (generic kernels, any 64-bit value): tab[k*256 + b] = crc(0, b << 8k).
// Chunk layout (tile kernels): 11/11/10-bit chunks aligned to each 32-bit
// word, chunk k covers bits [kShift[k], kShift[k] + width) and has a
// 2048-entry table at tab[k*2048].  Three lookups cover 32-bit positions, four
// cover 43 bits.  The byte offset (chunk << 2) of every chunk is formed on the
// FMA pipe by integer multiplies with launch-constant (opaque) powers of two,
// so the CRC costs one LOP3 per word on the ALU pipe instead of one PRMT per
// byte.

// chunk k covers bits [chunk_shift(k), chunk_shift(k) + chunk_width(k)): 0, 11, 22, 32, 43, 54
__host__ __device__ __forceinline__ uint32_t chunk_shift(int k) { return 32u * (k / 3) + 11u * (k % 3); }
__host__ __device__ __forceinline__ uint32_t chunk_width(int k) { return (k % 3 == 2) ? 10u : 11u; }

__device__ __forceinline__ void build_byte_tables(uint32_t *tab, int nb, uint32_t k0) {
    for (int e = threadIdx.x; e < nb * 256; e += blockDim.x) {
        const int k = e >> 8, b = e & 255;
        tab[e] = crc32c_u64_bitwise(0u, (uint64_t)b << (8 * k)) ^ (k == 0 ? k0 : 0u);
    }
}

__device__ __forceinline__ void build_chunk_tables(uint32_t *tab, int nc, uint32_t k0, int words = 1 << 30) {
    for (int e = threadIdx.x; e < nc * 2048 && e < words; e += blockDim.x) {
        const int k = e >> 11, x = e & 2047;
        uint32_t v = 0;
        if ((uint32_t)x < (1u << chunk_width(k)))
            v = crc32c_u64_bitwise(0u, (uint64_t)x << chunk_shift(k)) ^ (k == 0 ? k0 : 0u);
        tab[e] = v;
    }
}

// Seed-free chunk tables (k0 = 0) by CRC linearity: crc(0, x << s) is the
// XOR of crc(0, 1 << (s + j)) over the set bits j of x, so the 64 single-bit
// values are computed once (bitwise) and every entry costs <= 11 XORs -- for
// kernels with many short-lived CTAs.  bits: 64 words of shared scratch.
__device__ __forceinline__ void build_chunk_tables_linear(uint32_t *tab, int nc, uint32_t *bits, uint32_t k0 = 0u,
                                                          int words = 1 << 30) {
    if (threadIdx.x < 64) bits[threadIdx.x] = crc32c_u64_bitwise(0u, 1ull << threadIdx.x);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * 2048 && e < words; e += blockDim.x) {
        const int k = e >> 11;
        uint32_t x = (uint32_t)(e & 2047), v = 0;
        if (x < (1u << chunk_width(k))) {
            const uint32_t *bk = bits + chunk_shift(k);
            while (x) {
                const int j = __ffs(x) - 1;
                v ^= bk[j];
                x &= x - 1;
            }
            if (k == 0) v ^= k0;  // the seed's crc(s0, 0), folded into table 0
        }
        tab[e] = v;
    }
}

// Shared-space (32-bit) addressing: the tables are reached through a
// shared-window address kept in a register, so the compiler does not
// rematerialise the generic->shared conversion inside the loop.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint16_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u64(uint32_t addr, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" :: "r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void sts_u64_if(bool pred, uint32_t addr, uint64_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u64 [%1], %2;\n\t}"
                 :: "r"((unsigned)pred), "r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void sts_u32_if(bool pred, uint32_t addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u32 [%1], %2;\n\t}"
                 :: "r"((unsigned)pred), "r"(addr), "r"(v) : "memory");
}
template <class T>
__device__ __forceinline__ void sts_t_if(bool pred, uint32_t addr, T v) {
    if constexpr (sizeof(T) == 4) sts_u32_if(pred, addr, (uint32_t)v);
    else sts_u64_if(pred, addr, (uint64_t)v);
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" :: "r"(addr), "h"(v) : "memory");
}
// 32 bytes (two edge rows) with one streaming store (sm_100: STG.256); the
// address must be 32-byte aligned.
__device__ __forceinline__ void stcs_256(void *ptr, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
// Loop-invariant value the compiler must keep in a register (it would
// otherwise rematerialise shared-window bases inside the hot loop).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
template <class T>
__device__ __forceinline__ T lds_t(uint32_t addr) {
    if constexpr (sizeof(T) == 4) return (T)lds_u32(addr);
    else return (T)lds_u64(addr);
}
template <class T>
__device__ __forceinline__ void sts_t(uint32_t addr, T v) {
    if constexpr (sizeof(T) == 4) sts_u32(addr, (uint32_t)v);
    else sts_u64(addr, (uint64_t)v);
}

template <int NB>
__device__ __forceinline__ uint32_t crc_bytes(uint32_t tab, uint64_t w) {
    const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const uint32_t b = __byte_perm(k < 4 ? lo : hi, 0u, 0x4440u | (k & 3));
        c ^= lds_u32(tab + (k * 256 + b) * 4);
    }
    return c;
}

// crc of the three chunks of one 32-bit word, tables at t, t+8K, t+16K
// Byte offsets of the three 11/11/10-bit chunks of x (shift + mask on the
// ALU pipe: the FMA-heavy pipe that would take IMAD forms is the busier one).
__device__ __forceinline__ uint32_t crc_word3(uint32_t t, uint32_t x) {
#if PARBA_ROT
    const uint32_t o0 = __funnelshift_l(x, x, 2) & 0x1ffcu;   // rotate: SHF on the ALU
#else
    const uint32_t o0 = (x << 2) & 0x1ffcu;   // (x & 0x7ff) << 2
#endif
    const uint32_t o1 = (x >> 9) & 0x1ffcu;   // ((x >> 11) & 0x7ff) << 2
    const uint32_t o2 = (x >> 20) & 0xffcu;   // (x >> 22) << 2
    return lds_u32(t + o0) ^ lds_u32(t + 8192 + o1) ^ lds_u32(t + 16384 + o2);
}

template <int NC>
__device__ __forceinline__ uint32_t crc_chunks(uint32_t tab, uint64_t w) {
    uint32_t c = crc_word3(tab, (uint32_t)w);
    if constexpr (NC > 3) {
        const uint32_t hi = (uint32_t)(w >> 32);
        c ^= lds_u32(tab + 3 * 8192 + ((hi << 2) & 0x1ffcu));
        if constexpr (NC > 4) c ^= lds_u32(tab + 4 * 8192 + ((hi >> 9) & 0x1ffcu));
        if constexpr (NC > 5) c ^= lds_u32(tab + 5 * 8192 + ((hi >> 20) & 0xffcu));
    }
    return c;
}

// ---------------------------------------------------------------------------
// Hash policies.  R is the chain-value type (u32 when every position < 2^32).
// probe(tab, r) = h(r); from_crc(c0, r) finishes h from c0 = crc(s0, r).

// Tile kernels: chunk tables; NC = 2 (every r < 2^31; 3 tables), 3 (<= kR32Max,
// just below 2^32), 4 (< 2^43), 5 (< 2^52), 6 (any).
template <int NC>
struct HashCrc {
    static constexpr bool kHasCrc = true;
    static constexpr int kChunks = NC < 3 ? 3 : NC;
    static constexpr bool kNarrow = NC <= 3;
    static constexpr bool kR31 = NC == 2;
    static constexpr bool kPack = NC <= 5;       // every value < 2^52
    // 2048 entries per table; the last table of the 3-table (32-bit) layout
    // holds a 10-bit chunk, so it is 1024 entries
    static constexpr int kTableWords = kChunks == 3 ? 2 * 2048 + 1024 : kChunks * 2048;
    using R = typename std::conditional<kNarrow, uint32_t, uint64_t>::type;
    __device__ __forceinline__ static void build(uint32_t *tab, uint32_t k0) {
        build_chunk_tables(tab, kChunks, k0, kTableWords);
    }
    // the same tables from the 64 single-bit CRCs (bits: 64 words of shared
    // scratch; includes a __syncthreads): <= 11 XORs per entry instead of a
    // 64-step bitwise CRC
    __device__ __forceinline__ static void build_linear(uint32_t *tab, uint32_t *bits, uint32_t k0) {
        build_chunk_tables_linear(tab, kChunks, bits, k0, kTableWords);
    }
    __device__ __forceinline__ static R from_crc(uint32_t c0, R r, const DevParams &p) {
        if constexpr (NC == 2) return mod_fp31(c0, c0 ^ p.k01, r);
        else if constexpr (kNarrow && PARBA_R32) {
            const double rd = u32_to_f64(r);
            return mod_fp32_y(c0, c0 ^ p.k01, r, rd, recip_approx(rd));
        } else if constexpr (kNarrow) return mod_fp<R>(c0, c0 ^ p.k01, u32_to_f64(r));
        else if constexpr (NC <= 5) return mod_fp<R>(c0, c0 ^ p.k01, r_to_f64w(r));
        else return mod_int(c0, c0 ^ p.k01, r);
    }
    // Same, with rd = (double)r and y ~ 1/r (relative error < 2^-34) supplied
    // by the caller (first probes of a tile: series around the tile's centre).
    static constexpr bool kHasRy = NC <= 5;
    __device__ __forceinline__ static R from_crc_ry(uint32_t c0, R r, double rd, double y,
                                                    const DevParams &p) {
        if constexpr (NC == 2) return mod_fp31_y(c0, c0 ^ p.k01, r, rd, y);
        else if constexpr (kNarrow && PARBA_R32) return mod_fp32_y(c0, c0 ^ p.k01, r, rd, y);
        else return mod_fp_y<R>(c0, c0 ^ p.k01, rd, y);
    }
    // One-stage remainder (mod_fp31_y1 / mod_fp_y1w) for first probes of
    // tiles with 2*base >= kOneStageMin (every r >= 2^28): needs no rd
    static constexpr bool kHasRy1 = PARBA_ONESTAGE && (NC <= 3 || (NC <= 5 && PARBA_ONESTAGE_WIDE));
    // 4- and 5-chunk store kernels take it too (wide store +1.4%; the window -0.55%)
    static constexpr bool kHasRy1Store = PARBA_ONESTAGE && NC <= 5 && PARBA_ONESTAGE_WIDE_STORE;
    __device__ __forceinline__ static R from_crc_ry1(uint32_t c0, R r, double y, const DevParams &p) {
        if constexpr (NC == 2) return mod_fp31_y1(c0, c0 ^ p.k01, r, y);
        else return (R)mod_fp_y1w(c0, c0 ^ p.k01, (uint64_t)r, y);
    }
    __device__ __forceinline__ static uint32_t crc(uint32_t tab, uint64_t w, const DevParams &p) {
        return crc_chunks<kChunks>(tab, w);
    }
    __device__ __forceinline__ static R probe(uint32_t tab, R r, const DevParams &p) {
        return from_crc(crc(tab, r, p), r, p);
    }
};

// Generic kernels: byte tables, any 64-bit value.
struct HashCrcBytes {
    static constexpr bool kHasCrc = true;
    static constexpr bool kHasRy = false;
    template <class T>
    __device__ __forceinline__ static T from_crc_ry(uint32_t, T r, double, double, const DevParams &) { return r; }
    static constexpr bool kHasRy1 = false;
    static constexpr bool kHasRy1Store = false;
    template <class T>
    __device__ __forceinline__ static T from_crc_ry1(uint32_t, T r, double, const DevParams &) { return r; }
    static constexpr bool kNarrow = false;
    static constexpr bool kR31 = false;
    static constexpr bool kPack = false;
    static constexpr int kTableWords = 8 * 256;
    using R = uint64_t;
    __device__ __forceinline__ static void build(uint32_t *tab, uint32_t k0) { build_byte_tables(tab, 8, k0); }
    __device__ __forceinline__ static R probe(uint32_t tab, R r, const DevParams &p) {
        const uint32_t c0 = crc_bytes<8>(tab, r);
        return mod_int(c0, c0 ^ p.k01, r);
    }
};

template <bool NARROW>
struct HashSimple {
    static constexpr bool kHasCrc = false;
    static constexpr bool kHasRy = false;
    template <class T>
    __device__ __forceinline__ static T from_crc_ry(uint32_t, T r, double, double, const DevParams &) { return r; }
    static constexpr bool kHasRy1 = false;
    static constexpr bool kHasRy1Store = false;
    template <class T>
    __device__ __forceinline__ static T from_crc_ry1(uint32_t, T r, double, const DevParams &) { return r; }
    static constexpr bool kNarrow = NARROW;
    static constexpr bool kR31 = false;
    static constexpr bool kPack = NARROW;
    static constexpr int kTableWords = 0;
    using R = typename std::conditional<NARROW, uint32_t, uint64_t>::type;
    __device__ __forceinline__ static void build(uint32_t *, uint32_t) {}
    __device__ __forceinline__ static R probe(uint32_t, R r, const DevParams &p) {
        return (R)__umul64hi((uint64_t)r * p.mult, (uint64_t)r);
    }
};

// Full-warp ballot (callers guarantee convergence).
__device__ __forceinline__ unsigned ballot_all(bool pred) {
    unsigned m;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tvote.sync.ballot.b32 %0, q, 0xffffffff;\n\t}"
                 : "=r"(m) : "r"((unsigned)pred));
    return m;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace parba
