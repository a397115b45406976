// Full degree histogram by partition (SURVEY.md §8 row a, C4; the reference
// counts with `counts[v] += 1` per endpoint, analytics.py:44-48).
//
// Direct `atomicAdd(counts + target, 1)` into an n-word array runs at the L2
// atomic rate (~4.3e10/s on B200) no matter where the array lives.  The
// partitioned pass replaces it with shared-memory atomics:
//   1. tile_kernel<kTargets> appends every finished target (u32) to its
//      warp's region of a scratch buffer (UINT32_MAX = empty slot);
//   2. bucket_hist_kernel: per-CTA histogram of bucket = target >> shift
//      (nb <= kHistBuckets buckets), written bucket-major so one exclusive
//      scan gives every (bucket, CTA) its output offset;
//   3. bucket_scatter_kernel: each CTA re-reads its span in sub-tiles,
//      sorts a sub-tile by bucket in shared memory and writes the bucket
//      runs contiguously (no global atomics);
//   4. slice_count_kernel: one CTA per (bucket, 2^15-node slice) counts its
//      bucket's entries of that slice in shared memory and adds them to the
//      counts it owns exclusively (plain coalesced read-modify-write).
// HBM traffic per target: 4 B written + 3 x 4 B read + 4 B written; the
// bucket reads of step 4 repeat once per slice of the bucket (<= 8) and are
// served by L2 because a bucket's slices run side by side.
#pragma once
#include <cstdint>

namespace parba {

constexpr int kHistBuckets = 1024;          // level-1 buckets (max)
constexpr int kSliceLg = 15;                // level-2 slice: 2^15 counters
constexpr int kSliceNodes = 1 << kSliceLg;  // 128 KB of u32 in shared memory
constexpr int kMaxSliceLgPerBucket = 3;     // <= 8 slices per bucket
constexpr int kHistThreads = 1024;
constexpr int kScatterTile = 8192;          // entries per sorted sub-tile
constexpr int kScatterPer = kScatterTile / kHistThreads;
constexpr uint32_t kEmptyTarget = 0xffffffffu;

__device__ __forceinline__ uint4 ld_stream4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Step 2: H[b * gridDim.x + blk] = entries of CTA blk's span in bucket b.
// len and span are multiples of 4; t is 16-byte aligned.
__global__ void __launch_bounds__(kHistThreads) bucket_hist_kernel(const uint32_t *__restrict__ t, uint64_t len,
                                                                   uint64_t span, uint32_t n, int shift, int nb,
                                                                   uint32_t *__restrict__ H) {
    __shared__ uint32_t h[kHistBuckets];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const uint64_t s0 = (uint64_t)blockIdx.x * span;
    const uint64_t s1 = s0 + span < len ? s0 + span : len;
    const uint4 *t4 = reinterpret_cast<const uint4 *>(t + s0);
    const uint64_t n4 = s1 > s0 ? (s1 - s0) / 4 : 0;
    for (uint64_t k = threadIdx.x; k < n4; k += blockDim.x) {
        const uint4 v = __ldg(t4 + k);  // kept in L2 for the scatter re-read
        if (v.x < n) atomicAdd(&h[v.x >> shift], 1u);
        if (v.y < n) atomicAdd(&h[v.y >> shift], 1u);
        if (v.z < n) atomicAdd(&h[v.z >> shift], 1u);
        if (v.w < n) atomicAdd(&h[v.w >> shift], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) H[(uint64_t)b * gridDim.x + blockIdx.x] = h[b];
}

// Block-wide exclusive scan of x (one value per thread, kHistThreads threads).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *warp_sums) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sums[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t s = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    return inc - x + (w > 0 ? warp_sums[w - 1] : 0u);
}

// Step 3: O = exclusive scan of H (bucket-major).  CTA blk writes its
// bucket-b entries to out[O[b * gridDim.x + blk] ...] in sub-tile order.
__global__ void __launch_bounds__(kHistThreads) bucket_scatter_kernel(const uint32_t *__restrict__ t, uint64_t len,
                                                                      uint64_t span, uint32_t n, int shift, int nb,
                                                                      const uint32_t *__restrict__ O,
                                                                      uint32_t *__restrict__ out) {
    __shared__ uint32_t cur[kHistBuckets];    // next output position per bucket
    __shared__ uint32_t cnt[kHistBuckets];    // sub-tile entries per bucket
    __shared__ uint32_t start[kHistBuckets];  // sub-tile run start per bucket
    __shared__ uint32_t sorted[kScatterTile];
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t total_s;
    for (int b = threadIdx.x; b < kHistBuckets; b += blockDim.x)
        cur[b] = b < nb ? O[(uint64_t)b * gridDim.x + blockIdx.x] : 0u;
    const uint64_t s0 = (uint64_t)blockIdx.x * span;
    const uint64_t s1 = s0 + span < len ? s0 + span : len;
    for (uint64_t base = s0; base < s1; base += kScatterTile) {
        for (int b = threadIdx.x; b < kHistBuckets; b += blockDim.x) cnt[b] = 0;
        __syncthreads();
        uint32_t v[kScatterPer], rk[kScatterPer];
        // coalesced: thread i takes 16-byte words i and i + kHistThreads
#pragma unroll
        for (int h = 0; h < kScatterPer / 4; ++h) {
            const uint64_t e = base + 4ull * (threadIdx.x + (uint64_t)h * kHistThreads);
            uint4 w = make_uint4(kEmptyTarget, kEmptyTarget, kEmptyTarget, kEmptyTarget);
            if (e < s1) w = ld_stream4(reinterpret_cast<const uint4 *>(t + e));
            v[4 * h] = w.x;
            v[4 * h + 1] = w.y;
            v[4 * h + 2] = w.z;
            v[4 * h + 3] = w.w;
        }
#pragma unroll
        for (int k = 0; k < kScatterPer; ++k)
            if (v[k] < n) rk[k] = atomicAdd(&cnt[v[k] >> shift], 1u);
        __syncthreads();
        const uint32_t c = cnt[threadIdx.x];  // kHistThreads == kHistBuckets
        const uint32_t ex = block_exclusive_scan(c, warp_sums);
        start[threadIdx.x] = ex;
        if (threadIdx.x == kHistThreads - 1) total_s = ex + c;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kScatterPer; ++k)
            if (v[k] < n) sorted[start[v[k] >> shift] + rk[k]] = v[k];
        __syncthreads();
        const uint32_t total = total_s;
        for (uint32_t k = threadIdx.x; k < total; k += blockDim.x) {
            const uint32_t x = sorted[k];
            const uint32_t b = x >> shift;
            out[cur[b] + (k - start[b])] = x;
        }
        __syncthreads();
        cur[threadIdx.x] += c;
    }
}

// Step 4: CTA (b, s) counts bucket b's entries of slice s (nodes
// (b << shift) + (s << kSliceLg) + [0, 2^kSliceLg)) and adds them to counts.
// Bucket b's entries are sorted[O[b * nblk] .. O[(b + 1) * nblk]) (the last
// bucket ends at O[last] + H[last]).
__global__ void __launch_bounds__(kHistThreads) slice_count_kernel(const uint32_t *__restrict__ sorted,
                                                                   const uint32_t *__restrict__ O,
                                                                   const uint32_t *__restrict__ H, uint32_t nblk,
                                                                   int nb, uint32_t n, int shift, int spb_lg,
                                                                   uint32_t *__restrict__ counts) {
    extern __shared__ uint32_t c[];
    const uint32_t b = blockIdx.x >> spb_lg;
    const uint32_t s = blockIdx.x & ((1u << spb_lg) - 1);
    for (int k = threadIdx.x; k < kSliceNodes; k += blockDim.x) c[k] = 0;
    __syncthreads();
    const uint64_t last = (uint64_t)nb * nblk - 1;
    const uint32_t e0 = O[(uint64_t)b * nblk];
    const uint32_t e1 = (int)b + 1 < nb ? O[(uint64_t)(b + 1) * nblk] : O[last] + H[last];
    const uint32_t smask = (1u << spb_lg) - 1;
    for (uint32_t k = e0 + threadIdx.x; k < e1; k += blockDim.x) {
        const uint32_t x = __ldg(sorted + k);
        if (((x >> kSliceLg) & smask) == s) atomicAdd(&c[x & (kSliceNodes - 1)], 1u);
    }
    __syncthreads();
    const uint64_t v0 = ((uint64_t)b << shift) + ((uint64_t)s << kSliceLg);
    for (int k = threadIdx.x; k < kSliceNodes; k += blockDim.x) {
        const uint64_t v = v0 + k;
        if (v < n && c[k]) counts[v] += c[k];
    }
}

}  // namespace parba
