// parba_device.cuh -- device-side building blocks of the B200 hot path.
//
//   crc0<NB>(w)   CRC32-C of one 64-bit word with zero seed, w < 2^(8*NB):
//                 slicing tables tab[k][b] = crc(0, b << 8k) in shared memory,
//                 one lookup per significant byte (4 for 2m <= 2^32, 5 for the
//                 paper-scale 1e11-edge graph).  Byte extraction is one PRMT
//                 (ALU pipe) and the scaled address one IMAD (FMA pipe).
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
    Magic32 div32;         // by d (narrow: positions < 2^32)
    uint64_t win_rlim;     // window mode: generated target < K  <=>  r < win_rlim
    uint32_t win_rlim32;   // min(win_rlim, 2^32 - 1) for narrow launches
    uint64_t K;
};

// Closed forms (generator.py:157-169): source of edge i, target of terminal r.
template <bool NARROW, bool SEED>
__device__ __forceinline__ uint64_t source_of(uint64_t i, const DevParams &p) {
    if constexpr (NARROW) {
        if constexpr (SEED) return (uint64_t)magic_div32((uint32_t)(i - p.m0), p.div32) + p.n0;
        else return (uint64_t)magic_div32((uint32_t)i, p.div32);
    } else {
        if constexpr (SEED) return magic_div(i - p.m0, p.div64) + p.n0;
        else return magic_div(i, p.div64);
    }
}
template <bool NARROW, bool SEED>
__device__ __forceinline__ uint64_t target_of(uint64_t r, const DevParams &p) {
    if constexpr (SEED) {
        if (r < p.stop) return __ldg(p.seed + r);
    }
    return source_of<NARROW, SEED>(r >> 1, p);
}

// ---------------------------------------------------------------------------
// Exact remainder.

__device__ __forceinline__ double u32_to_f64(uint32_t x) {
    return __hiloint2double(0x43300000, (int)x) - 0x1p52;
}
__device__ __forceinline__ double u52_to_f64(uint64_t x) {  // x < 2^52
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 0x1p52;
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
__device__ __forceinline__ R mod_fp(uint32_t hhi, uint32_t hlo, double rd) {
    const double y = recip_approx(rd);
    const double ha = u32_to_f64(hhi);
    const double hl = u32_to_f64(hlo);
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
    const uint32_t qb = (uint32_t)__double2loint(fma(u64_halves_to_f64((uint32_t)x, hlo), y, 0x1p52));
    int64_t t = (int64_t)(v - (uint64_t)qb * r);       // in [-r, r): fits for r <= 2^63
    t += (t < 0) ? (int64_t)r : 0;
    return (uint64_t)t;
}

// ---------------------------------------------------------------------------
// Byte-sliced CRC tables in shared memory: tab[k][b] = crc(0, b << 8k).

template <int NB>
struct CrcTables {
    uint32_t t[NB][256];
};

// Table 0 carries k0 = crc(s0, 0): every crc0() XORs exactly one table-0
// entry, so crc0() returns crc(s0, w) directly (CRC linearity).
template <int NB>
__device__ __forceinline__ void build_crc_tables(CrcTables<NB> &s, uint32_t k0) {
    for (int e = threadIdx.x; e < NB * 256; e += blockDim.x) {
        const int k = e >> 8, b = e & 255;
        s.t[k][b] = crc32c_u64_bitwise(0u, (uint64_t)b << (8 * k)) ^ (k == 0 ? k0 : 0u);
    }
}

template <int NB>
__device__ __forceinline__ uint32_t crc0(const CrcTables<NB> &s, uint64_t w) {
    const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const uint32_t b = __byte_perm(k < 4 ? lo : hi, 0u, 0x4440u | (k & 3));
        c ^= s.t[k][b];
    }
    return c;
}

// ---------------------------------------------------------------------------
// Hash policies.  R is the chain-value type (u32 when every position < 2^32).

template <int NB>
struct HashCrc {
    static constexpr bool kHasCrc = true;
    static constexpr bool kNarrow = NB <= 4;
    static constexpr int kTables = NB;
    using R = typename std::conditional<kNarrow, uint32_t, uint64_t>::type;
    // c0 = crc(s0, r) (k0 already folded into table 0); crc(s1, r) = c0 ^ k01.
    __device__ __forceinline__ static R from_crc(uint32_t c0, R r, const DevParams &p) {
        if constexpr (kNarrow) return mod_fp<R>(c0, c0 ^ p.k01, u32_to_f64(r));
        else if constexpr (NB * 8 <= 52) return mod_fp<R>(c0, c0 ^ p.k01, u52_to_f64(r));
        else return mod_int(c0, c0 ^ p.k01, r);
    }
    __device__ __forceinline__ static R probe(const CrcTables<NB> &s, R r, const DevParams &p) {
        return from_crc(crc0<NB>(s, r), r, p);
    }
};

template <bool NARROW>
struct HashSimple {
    static constexpr bool kHasCrc = false;
    static constexpr bool kNarrow = NARROW;
    static constexpr int kTables = 1;
    using R = typename std::conditional<NARROW, uint32_t, uint64_t>::type;
    __device__ __forceinline__ static R probe(const CrcTables<1> &, R r, const DevParams &p) {
        return (R)__umul64hi((uint64_t)r * p.mult, (uint64_t)r);
    }
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace parba
