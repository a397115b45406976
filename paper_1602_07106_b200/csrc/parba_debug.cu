// parba_debug.cu -- direct access to the exact-remainder routines every tile
// kernel uses for h % r (_kernels.py:32-42; hashing.py:119-125), so tests can
// pin them against exact integer division on arbitrary and adversarial
// (hhi, hlo, r) -- not only on the values a CRC happens to produce.
//
//   PARBA_MOD_FP31       mod_fp31 (HashCrc<2>: r < 2^31)
//   PARBA_MOD_FP_NARROW  mod_fp<u32> with I2F of r (r < 2^32; HashCrc<3> before mod_fp32_y)
//   PARBA_MOD_FP32       mod_fp32_y (HashCrc<3>: r <= kR32Max = 0xF0000000), and its
//                        series form PARBA_MOD_FP32_SERIES
//   PARBA_MOD_FP_WIDE    mod_fp<u64> with the wide conversion (HashCrc<4,5>: r < 2^52)
//   PARBA_MOD_INT        mod_int (HashCrc<6>, HashCrcBytes: any r >= 1)
//   PARBA_MOD_*_SERIES   the same remainders with 1/r taken from phase 1's
//                        per-tile reciprocal series (tile_kernel, 2*base >= 2^27):
//                        element k plays lane-slot k % 8 of a lane whose centre
//                        is rc = r - (64*(k % 8) - 224).
//   PARBA_MOD_FP31_SERIES1  the series with phase 1's one-stage remainder
//                        (mod_fp31_y1: 2-chunk tiles with 2*base >= 2^28)
//   PARBA_MOD_FP_WIDE_SERIES1  the same for 3- to 5-chunk tiles (mod_fp_y1w)
//   parba_debug_rcp_bound   the exact error bound of rcp.approx.ftz.f64
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/parba_b200.h"
#include "parba_common.h"

using namespace parba;
using namespace parba::host;

namespace {

__device__ __forceinline__ uint64_t eval_mod(int method, uint32_t hhi, uint32_t hlo, uint64_t r, int slot) {
    switch (method) {
        case PARBA_MOD_FP31: return mod_fp31(hhi, hlo, (uint32_t)r);
        case PARBA_MOD_FP_NARROW: return mod_fp<uint32_t>(hhi, hlo, u32_to_f64((uint32_t)r));
        case PARBA_MOD_FP_WIDE: return mod_fp<uint64_t>(hhi, hlo, r_to_f64w(r));
        case PARBA_MOD_INT: return mod_int(hhi, hlo, r);
        case PARBA_MOD_FP32: {
            const double rd = u32_to_f64((uint32_t)r);
            return mod_fp32_y(hhi, hlo, (uint32_t)r, rd, recip_approx(rd));
        }
        default: break;
    }
    // series: the lane's centre rc, c = 1/rc, y_k = c - (k - 3.5) * 64 c^2
    // (tile_kernel phase1, RY branch); r = rc + 64k - 224 exactly
    const double e = 64.0 * slot - 224.0;
    const double rc = u52_to_f64(r) - e;
    const double c = recip_approx(rc);
    const double s64 = 64.0 * c * c;
    const double y = fma(-(slot - 3.5), s64, c);
    const double rd = rc + e;
    switch (method) {
        case PARBA_MOD_FP31_SERIES1: return mod_fp31_y1(hhi, hlo, (uint32_t)r, y);
        case PARBA_MOD_FP_WIDE_SERIES1: return mod_fp_y1w(hhi, hlo, r, y);
        case PARBA_MOD_FP31_SERIES: return mod_fp31_y(hhi, hlo, (uint32_t)r, rd, y);
        case PARBA_MOD_FP_NARROW_SERIES: return mod_fp_y<uint32_t>(hhi, hlo, rd, y);
        case PARBA_MOD_FP32_SERIES: return mod_fp32_y(hhi, hlo, (uint32_t)r, rd, y);
        default: return mod_fp_y<uint64_t>(hhi, hlo, rd, y);
    }
}

__global__ void mod_eval_kernel(int method, const uint32_t *__restrict__ hhi, const uint32_t *__restrict__ hlo,
                                const uint64_t *__restrict__ r, uint64_t count, uint64_t *__restrict__ out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = eval_mod(method, hhi[k], hlo[k], r[k], (int)(k & 7));
}

__device__ __forceinline__ uint64_t splitmix(uint64_t &s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Random and adversarial (h, r) drawn on the device, checked against the
// compiler's exact u64 % (an ~80-instruction integer subroutine).
__global__ void mod_check_kernel(int method, uint64_t seed, uint64_t count, uint64_t rmin, uint64_t rmax,
                                 unsigned long long *bad, unsigned long long *first) {
    const int bmin = 64 - __clzll(rmin), bmax = 64 - __clzll(rmax);
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = seed ^ (k * 0xD1B54A32D192ED03ull);
        const uint64_t x0 = splitmix(s), x1 = splitmix(s), x2 = splitmix(s);
        // r: log-uniform bit length in [bits(rmin), bits(rmax)], clamped
        const int b = bmin + (int)(x0 % (uint64_t)(bmax - bmin + 1));
        uint64_t r = (b >= 64 ? x1 : (x1 & ((1ull << b) - 1))) | (1ull << (b - 1));
        r = r < rmin ? rmin : (r > rmax ? rmax : r);
        // h: uniform, or next to a multiple of r, or with an all-ones half
        uint64_t h = x2;
        const uint32_t kind = (uint32_t)(x0 >> 56) & 7u;
        if (kind == 1 || kind == 2) {
            const uint64_t q = x2 / r;  // h = q*r + {-1, 0, +1} (mod 2^64)
            h = q * r + (uint64_t)(int64_t)((int)(x0 >> 40) % 3 - 1);
        } else if (kind == 3) {
            h = x2 | 0xFFFFFFFF00000000ull;
        } else if (kind == 4) {
            h = x2 | 0x00000000FFFFFFFFull;
        } else if (kind == 5) {
            h = (x2 % r) + r * ((x0 >> 8) & 1);  // small h (< 2r)
        }
        const uint64_t want = h % r;
        const uint64_t got = eval_mod(method, (uint32_t)(h >> 32), (uint32_t)h, r, (int)(k & 7));
        if (got != want) {
            if (atomicAdd(bad, 1ull) == 0) {
                first[0] = h;
                first[1] = r;
                first[2] = got;
            }
        }
    }
}

bool method_ok(int m) { return m >= PARBA_MOD_FP31 && m <= PARBA_MOD_FP32_SERIES; }

// rcp.approx.ftz.f64 (MUFU.RCP64H) reads only the high word of its operand:
// for one high word (sign 0, biased exponent E, top 20 mantissa bits M) the
// result y0 is one value, and |y0*x - 1| over the 2^32 operands sharing that
// high word is largest at the two ends of the low word.  So the maximum over
// all 2^20 values of M at both ends is the exact bound of the instruction's
// relative error for exponent E (out[0]); out[1] is the same for the
// Newton-refined recip_approx at those operands.  Exponents E0 .. E0+ne-1.
__global__ void rcp_bound_kernel(int e0, int ne, unsigned long long *out) {
    double m0 = 0.0, m1 = 0.0;
    const uint32_t total = (uint32_t)ne << 21;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
        const uint32_t E = (uint32_t)e0 + (k >> 21), M = (k >> 1) & 0xFFFFFu, lo = (k & 1u) ? 0xFFFFFFFFu : 0u;
        const double x = __hiloint2double((int)((E << 20) | M), (int)lo);
        double y0;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
        m0 = fmax(m0, fabs(fma(y0, x, -1.0)));
        m1 = fmax(m1, fabs(fma(recip_approx(x), x, -1.0)));
    }
    // non-negative doubles order like their bit patterns
    atomicMax(out, (unsigned long long)__double_as_longlong(m0));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(m1));
}

}  // namespace

extern "C" {

int parba_debug_mod(int method, const uint32_t *hhi, const uint32_t *hlo, const uint64_t *r, uint64_t count,
                    uint64_t *out, void *stream) {
    if (!method_ok(method)) return fail(PARBA_EINVAL, "unknown remainder method %d", method);
    if (count == 0) return PARBA_OK;
    if (!hhi || !hlo || !r || !out) return fail(PARBA_EINVAL, "NULL buffer");
    mod_eval_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(method, hhi, hlo, r, count, out);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_debug_mod_check(int method, uint64_t seed, uint64_t count, uint64_t rmin, uint64_t rmax,
                          unsigned long long *mismatches, unsigned long long *first_bad, void *stream) {
    if (!method_ok(method)) return fail(PARBA_EINVAL, "unknown remainder method %d", method);
    if (rmin < 1 || rmax < rmin) return fail(PARBA_EINVAL, "need 1 <= rmin <= rmax");
    if (!mismatches || !first_bad) return fail(PARBA_EINVAL, "NULL buffer");
    if (count == 0) return PARBA_OK;
    mod_check_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(method, seed, count, rmin, rmax, mismatches,
                                                                   first_bad);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_debug_rcp_bound(int e0, int ne, double *out, void *stream) {
    if (e0 < 1 || ne < 1 || e0 + ne > 2047) return fail(PARBA_EINVAL, "exponents must lie in [1, 2046]");
    if (!out) return fail(PARBA_EINVAL, "NULL buffer");
    CUDA_TRY(cudaMemsetAsync(out, 0, 2 * sizeof(double), (cudaStream_t)stream));
    rcp_bound_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(e0, ne, (unsigned long long *)out);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

}  // extern "C"
