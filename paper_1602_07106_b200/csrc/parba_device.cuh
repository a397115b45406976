// parba_device.cuh -- device-side building blocks of the B200 hot path.
//
//   crc0(w)       CRC32-C of one 64-bit word with zero seed, from 5-bit chunk
//                 tables in shared memory (32 entries per table = exactly the
//                 32 smem banks, so every lookup is bank-conflict free).
//   h_crc(r)      the reference hash ((crc(s0,r)<<32) + crc(s1,r)) % r
//                 (hashing.py:119-125, _kernels.py:32-42) rewritten through
//                 CRC linearity: crc(s,w) = crc(s,0) ^ crc(0,w), so one table
//                 CRC per probe instead of two.
//   mod_u64(h,r)  exact h % r via an fp64 reciprocal estimate (the FP64 pipe
//                 is otherwise idle) and one integer correction; a rare slow
//                 path (r < 2^13 or a failed correction) uses the exact
//                 integer remainder.
//   h_simple(r)   umulhi((r*M) mod 2^64, r)  (hashing.py:128-138).
//   MagicDiv      division by the launch-constant d (source/target closed
//                 forms, generator.py:157-169) by multiply-high.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace parba {

constexpr uint32_t kCrcPoly = 0x82F63B78u;  // hashing.py:40 (reflected 0x1EDC6F41)
constexpr int kChunkBits = 5;
constexpr int kMaxChunks = 13;              // ceil(64 / 5)

// Bit-serial CRC32-C of one LE 64-bit word (host + device); used only to
// build tables and constants.
__host__ __device__ inline uint32_t crc32c_u64_bitwise(uint32_t seed, uint64_t word) {
    uint32_t c = seed;
    for (int b = 0; b < 64; ++b) {
        uint32_t bit = (c ^ (uint32_t)(word >> b)) & 1u;
        c = (c >> 1) ^ (kCrcPoly & (0u - bit));
    }
    return c;
}

// Branch-free unsigned 64-bit division by a runtime-invariant d >= 1
// (Granlund-Montgomery round-up variant).
struct MagicDiv {
    uint64_t mul;
    uint32_t sh1, sh2;
};

inline MagicDiv make_magic(uint64_t d) {
    MagicDiv m{};
    int l = 0;
    while (l < 64 && (1ull << l) < d) ++l;  // l = ceil(log2 d)
    // mul = floor(2^64 * (2^l - d) / d) + 1
    unsigned __int128 num = ((unsigned __int128)1 << 64) * (((unsigned __int128)1 << l) - d);
    m.mul = (uint64_t)(num / d) + 1;
    m.sh1 = l > 0 ? 1u : 0u;
    m.sh2 = l > 0 ? (uint32_t)(l - 1) : 0u;
    return m;
}

__device__ __forceinline__ uint64_t magic_div(uint64_t n, const MagicDiv &m) {
    uint64_t t = __umul64hi(m.mul, n);
    return (t + ((n - t) >> m.sh1)) >> m.sh2;
}

// Launch-constant description of one graph family (plain uniform-d mode).
struct DevParams {
    uint64_t n, d, n0, m0, m;
    uint64_t stop;         // 2*m0: chains stop when r < stop (seed region)
    uint64_t mult;         // SIMPLE multiplier
    uint32_t k0, k1;       // crc(s0,0), crc(s1,0)
    const uint64_t *seed;  // 2*m0 seed endpoints (device)
    MagicDiv divd;
    uint64_t win_lim;      // window mode: generated target < K  <=>  (r>>1) < win_lim
    uint64_t K;
};

// Closed forms (generator.py:157-169): source of edge i, target of terminal r.
__device__ __forceinline__ uint64_t source_of(uint64_t i, const DevParams &p) {
    return magic_div(i - p.m0, p.divd) + p.n0;
}
__device__ __forceinline__ uint64_t target_of(uint64_t r, const DevParams &p) {
    if (r < p.stop) return __ldg(p.seed + r);
    return magic_div((r >> 1) - p.m0, p.divd) + p.n0;
}

// ---------------------------------------------------------------------------
// Exact 64-bit remainder.

__device__ __forceinline__ double u64_to_f64_exact52(uint64_t x) {  // x < 2^52
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 0x1p52;
}

// h = hi:lo (two u32 halves) -> nearest double (one rounding).
__device__ __forceinline__ double u64_halves_to_f64(uint32_t hi, uint32_t lo) {
    double dh = __hiloint2double(0x45300000, (int)hi);  // 2^84 + hi*2^32
    double dl = __hiloint2double(0x43300000, (int)lo);  // 2^52 + lo
    return (dh - 0x1.00000001p84) + dl;                  // 2^84 + 2^52 exactly
}

template <bool kWide>
__device__ __forceinline__ uint64_t mod_u64(uint32_t hhi, uint32_t hlo, uint64_t r) {
    const uint64_t h = ((uint64_t)hhi << 32) | hlo;
    if (r < (1ull << 13)) return h % r;  // q would exceed 2^51: exact slow path (rare)
    double rd = kWide ? __ull2double_rn(r) : u64_to_f64_exact52(r);
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rd));
    double e = fma(-rd, y, 1.0);
    y = fma(y, e, y);
    e = fma(-rd, y, 1.0);
    y = fma(y, e, y);
    double qd = u64_halves_to_f64(hhi, hlo) * y;   // ~ h / r, |err| < 2 for r >= 2^13
    uint64_t q = (uint64_t)__double_as_longlong(qd + 0x1p52) & 0x000FFFFFFFFFFFFFull;
    uint64_t t = h - q * r;                        // exact h mod r up to +-r
    if ((int64_t)t < 0) t += r;
    else if (t >= r) t -= r;
    if (t >= r) t = h % r;                         // estimate off by > 1: exact fallback
    return t;
}

// ---------------------------------------------------------------------------
// Shared-memory CRC tables: tab[k][x] = crc(0, x << 5k).

struct CrcTables {
    uint32_t t[kMaxChunks][32];
};

__device__ __forceinline__ void build_crc_tables(CrcTables &s) {
    for (int e = threadIdx.x; e < kMaxChunks * 32; e += blockDim.x) {
        int k = e >> 5, x = e & 31;
        s.t[k][x] = crc32c_u64_bitwise(0u, (uint64_t)x << (kChunkBits * k));
    }
}

// crc(0, w) for w < 2^(5*NCH).
template <int NCH>
__device__ __forceinline__ uint32_t crc0(const CrcTables &s, uint64_t w) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < NCH; ++k) c ^= s.t[k][(uint32_t)(w >> (kChunkBits * k)) & 31u];
    return c;
}

// ---------------------------------------------------------------------------
// Hash policies.  probe(r) = h(r); first(...) = h(2i+1) given crc(0,2i+1).

template <int NCH>
struct HashCrc {
    static constexpr bool kWide = (NCH * kChunkBits) > 52;
    static constexpr bool kHasCrc = true;
    __device__ __forceinline__ static uint64_t from_crc(uint32_t c, uint64_t r, const DevParams &p) {
        return mod_u64<kWide>(c ^ p.k0, c ^ p.k1, r);
    }
    __device__ __forceinline__ static uint64_t probe(const CrcTables &s, uint64_t r, const DevParams &p) {
        return from_crc(crc0<NCH>(s, r), r, p);
    }
};

struct HashSimple {
    static constexpr bool kHasCrc = false;
    __device__ __forceinline__ static uint64_t probe(const CrcTables &, uint64_t r, const DevParams &p) {
        return __umul64hi(r * p.mult, r);
    }
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace parba
