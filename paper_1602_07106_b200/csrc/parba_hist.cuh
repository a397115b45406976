// Full degree histogram by partition (SURVEY.md §8 row a, C4; the reference
// counts with `counts[v] += 1` per endpoint, analytics.py:44-48).
//
// Direct `atomicAdd(counts + target, 1)` into an n-word array runs at the L2
// atomic rate (~4.3e10/s on B200) no matter where the array lives.  The
// partitioned pass replaces it with shared-memory atomics:
//   1. tile_kernel<kTargets> appends every finished target (u32) to its
//      warp's region of a scratch buffer (UINT32_MAX = empty slot) and keeps
//      a per-CTA histogram of bucket = target >> shift (nb <= kHistBuckets),
//      written bucket-major so one exclusive scan gives every (bucket, CTA)
//      its output offset;
//   2. bucket_scatter_kernel: one CTA per tile CTA re-reads that CTA's
//      region in sub-tiles, sorts a sub-tile by bucket in shared memory and
//      writes the bucket runs contiguously (no global atomics);
//   3. slice_count_kernel: one CTA per (bucket chunk, 2^15-node slice)
//      counts the chunk's entries of that slice in shared memory and adds
//      them to counts (plain read-modify-write when it owns the bucket).
// HBM traffic per target: 4 B written, 4 B read + 4 B written by the
// scatter, 4 B read by the count; the count's reads repeat once per slice of
// a bucket (<= 8) and are served by L2 because those CTAs run side by side.
#pragma once
#include <cstdint>

namespace parba {

constexpr int kSliceLg = 15;                // level-2 slice: 2^15 counters
constexpr int kSliceNodes = 1 << kSliceLg;  // 128 KB of u32 in shared memory
constexpr int kMaxSliceLgPerBucket = 3;     // <= 8 slices per bucket
constexpr uint32_t kSliceMax = 57344;       // one-slice buckets (any width): 224 KB of u32
constexpr int kHistThreads = 1024;
#ifndef PARBA_SCATTER_TILE
#define PARBA_SCATTER_TILE 16384
#endif
#ifndef PARBA_SCATTER_THREADS
#define PARBA_SCATTER_THREADS 1024
#endif
constexpr int kScatterThreads = PARBA_SCATTER_THREADS;
#ifndef PARBA_COUNT_LOADS
#define PARBA_COUNT_LOADS 8  // 16-byte loads in flight per thread in the slice count
#endif
#ifndef PARBA_FLUSH_UNROLL
#define PARBA_FLUSH_UNROLL 4
#endif
constexpr int kScatterTile = PARBA_SCATTER_TILE;  // entries per sorted sub-tile (dynamic smem)
constexpr int kScatterSmem = (4 * kHistBuckets + kScatterTile) * 4;
constexpr uint32_t kEmptyTarget = 0xffffffffu;

__device__ __forceinline__ uint4 ld_stream4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Generic input (edge rows already in memory, e.g. the option-flag paths):
// CTA c copies the targets (.y) of rows [c * span, (c + 1) * span) that are
// < K into slots of the same index (others and slots past n_rows: empty)
// and writes its bucket histogram H[b * gridDim.x + c] -- the layout the
// targets sink produces, with one warp group per CTA.
__global__ void __launch_bounds__(1024) rows_targets_kernel(const ulonglong2 *__restrict__ rows, uint64_t n_rows,
                                                            uint64_t span, uint64_t K, int shift, int nb,
                                                            uint32_t *__restrict__ t32, uint32_t *__restrict__ H) {
    __shared__ uint32_t h[kHistBucketsMax];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const uint64_t s0 = (uint64_t)blockIdx.x * span;
    for (uint64_t k = s0 + threadIdx.x; k < s0 + span; k += blockDim.x) {
        uint32_t v = kEmptyTarget;
        if (k < n_rows) {
            const uint64_t tg = __ldg(&rows[k].y);
            if (tg < K) {
                v = (uint32_t)tg;
                atomicAdd(&h[v >> shift], 1u);
            }
        }
        t32[k] = v;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) H[(uint64_t)b * gridDim.x + blockIdx.x] = h[b];
}

// Block-wide exclusive scan of x (one value per thread, <= 1024 threads).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *warp_sums) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sums[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < nw ? warp_sums[lane] : 0u;
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

// Step 2: O = exclusive scan of H (bucket-major).  Scatter CTA c handles
// warp group c % groups of tile CTA c / groups: slots
// [(blk * wpc + w0) * capw, (blk * wpc + w1) * capw) with w0..w1 the group's
// warps, and writes its bucket-b entries to out[O[b * gridDim.x + c] ...] in
// sub-tile order.  One pass handles buckets [wb, wb + nbw) (nbw <=
// kHistBuckets) and skips the others.  T threads, kScatterTile entries per
// sub-tile.
// Strided input (nw > 0: the store-targets sink's tile-order slots): tile
// CTA c owns tiles k*nw + c*wpc + [0, wpc) for k = 0, 1, ... below ntiles,
// i.e. its k-th block of wpc*kTile entries starts at slot (k*nw + c*wpc)*kTile.
// OFF16: one-slice buckets of width bw < 2^16 -- each entry is written as
// its u16 offset in the bucket (target - bucket * bw), half the bytes of the
// scatter's writes and of the count's reads.
template <int T, bool OFF16 = false>
__global__ void __launch_bounds__(T, 1) bucket_scatter_kernel(const uint32_t *__restrict__ t, uint64_t len,
                                                           uint32_t wpc, uint32_t groups, uint64_t capw,
                                                           Magic32 bdiv, int wb, int nbw,
                                                           const uint32_t *__restrict__ O,
                                                           uint32_t *__restrict__ out, uint64_t nw,
                                                           uint64_t ntiles, uint32_t bw = 0, int tlg = 8) {
    const uint32_t kTile = 1u << tlg;  // strided input: edges per tile of the targets launch (256 or 512)
    constexpr int BPT = kHistBuckets / T;  // buckets per thread in the scan
    constexpr int PER = kScatterTile / T;  // entries per thread and sub-tile
    static_assert(BPT * T == kHistBuckets && PER % 4 == 0, "scatter shape");
    extern __shared__ uint32_t scatter_smem[];  // kScatterSmem bytes
    uint32_t *cur = scatter_smem;                  // next output position per bucket
    uint32_t *cnt = cur + kHistBuckets;            // sub-tile entries per bucket
    uint32_t *start = cnt + kHistBuckets;          // sub-tile run start per bucket
    uint32_t *delta = start + kHistBuckets;        // output position - sub-tile position
    uint32_t *sorted = delta + kHistBuckets;       // kScatterTile entries
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t total_s;
    const uint32_t c = blockIdx.x, blk = c / groups, g = c % groups;
    for (int b = threadIdx.x; b < kHistBuckets; b += T)
        cur[b] = b < nbw ? O[(uint64_t)(wb + b) * gridDim.x + c] : 0u;
    // an entry's bucket in this pass: (v >> shift) - wb, kept when < nbw
    // (empty slots, UINT32_MAX, land above every pass: buckets < 2^(32-shift) - 1)
    // (bucket = v / width: {1, shift} for a power-of-two width, else a
    // multiply-high -- exact for v < 2^31; empty slots map far above nbw)
    auto wbucket = [&](uint32_t v) -> uint32_t {
        return (uint32_t)(((uint64_t)v * bdiv.mul) >> bdiv.shift) - (uint32_t)wb;
    };
    const uint64_t c0 = (uint64_t)c * wpc;  // strided input: first tile of this CTA
    uint64_t s0 = ((uint64_t)blk * wpc + g * wpc / groups) * capw;
    const uint64_t e1 = ((uint64_t)blk * wpc + (g + 1) * wpc / groups) * capw;
    uint64_t s1 = e1 < len ? e1 : len;
    if (nw) {  // strided: logical entries [0, rounds * wpc * kTile) of this CTA (groups == 1)
        s0 = 0;
        s1 = ntiles > c0 ? (ntiles - c0 + nw - 1) / nw * wpc * kTile : 0;
    }
    // coalesced: thread i takes 16-byte words i, i + T, ... of a sub-tile; the
    // next sub-tile's loads are issued before this one is sorted
    uint4 nx[PER / 4];
    // strided input: logical entry e of this CTA -> block k = e / (wpc*kTile),
    // offset within the block; k by a float reciprocal of wpc on e / kTile
    // (< 2^24, the +1/2 margin keeps the rounding exact)
    const float inv_wpc = 1.0f / (float)wpc;
    auto load = [&](uint64_t base) {
#pragma unroll
        for (int h = 0; h < PER / 4; ++h) {
            const uint64_t e = base + 4ull * (threadIdx.x + (uint64_t)h * T);
            nx[h] = make_uint4(kEmptyTarget, kEmptyTarget, kEmptyTarget, kEmptyTarget);
            if (nw) {
                const uint32_t x = (uint32_t)(e >> tlg);  // logical tile of this CTA
                const uint32_t k = __float2uint_rz(__fmaf_rn((float)x, inv_wpc, 0.5f * inv_wpc));
                const uint64_t tile = (uint64_t)k * nw + c0 + (x - k * wpc);
                if (e < s1 && tile < ntiles)
                    nx[h] = ld_stream4(reinterpret_cast<const uint4 *>(t + tile * kTile + (e & (kTile - 1))));
            } else if (e < s1) {
                nx[h] = ld_stream4(reinterpret_cast<const uint4 *>(t + e));
            }
        }
    };
    load(s0);
    for (int b = threadIdx.x; b < kHistBuckets; b += T) cnt[b] = 0;
    __syncthreads();
    uint32_t v[PER], rk[PER];
    // rank of every entry of the sub-tile in nx within its bucket (shared
    // atomics on cnt), prefetching the sub-tile after it
    auto rank = [&]() {
#pragma unroll
        for (int h = 0; h < PER / 4; ++h) {
            v[4 * h] = nx[h].x;
            v[4 * h + 1] = nx[h].y;
            v[4 * h + 2] = nx[h].z;
            v[4 * h + 3] = nx[h].w;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (v[k] != kEmptyTarget && wbucket(v[k]) < (uint32_t)nbw) rk[k] = atomicAdd(&cnt[wbucket(v[k])], 1u);
    };
    if (s0 < s1) {
        rank();
        load(s0 + kScatterTile);
    }
    // five barriers per sub-tile: every shared array is rewritten only after
    // a barrier that its previous readers must have passed.  The next
    // sub-tile's ranks (cnt) are taken while this one's sorted runs are
    // written out (sorted, delta): disjoint arrays, so the two overlap.
    for (uint64_t base = s0; base < s1; base += kScatterTile) {
        __syncthreads();
        uint32_t cb[BPT], sum = 0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            cb[i] = cnt[threadIdx.x * BPT + i];
            cnt[threadIdx.x * BPT + i] = 0;  // ready for the next sub-tile
            sum += cb[i];
        }
        uint32_t ex = block_exclusive_scan(sum, warp_sums);
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            const int b = threadIdx.x * BPT + i;
            start[b] = ex;
            delta[b] = cur[b] - ex;  // output position of sorted[k] is delta[b] + k
            cur[b] += cb[i];
            ex += cb[i];
        }
        if (threadIdx.x == T - 1) total_s = ex;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (v[k] != kEmptyTarget && wbucket(v[k]) < (uint32_t)nbw) sorted[start[wbucket(v[k])] + rk[k]] = v[k];
        __syncthreads();
        const bool more = base + kScatterTile < s1;
        if (more) rank();
        const uint32_t total = total_s;
        for (uint32_t k = threadIdx.x; k < total; k += T) {
            const uint32_t x = sorted[k];
            const uint32_t b = wbucket(x);
            PARBA_CHECK(delta[b] + k < len);
            if constexpr (OFF16) {
                PARBA_CHECK(x - (wb + b) * bw < bw);
                reinterpret_cast<uint16_t *>(out)[delta[b] + k] = (uint16_t)(x - (wb + b) * bw);
            } else {
                out[delta[b] + k] = x;
            }
        }
        if (more) load(base + 2 * kScatterTile);
    }
}

// Step 3 plan: bucket sizes are skewed (node v draws ~ 1/sqrt(v) of the
// targets, so the lowest bucket holds several percent of all entries).  A
// bucket is cut into chunks of at most kCountChunk entries; items[] lists
// (bucket, chunk) pairs (bucket | chunk << kBucketBits).  One CTA of kHistThreads.
constexpr uint32_t kCountChunk = 1u << 21;

__device__ __forceinline__ void bucket_range(const uint32_t *O, const uint32_t *H, uint32_t nblk, int nb, uint32_t b,
                                             uint32_t &e0, uint32_t &e1) {
    const uint64_t last = (uint64_t)nb * nblk - 1;
    e0 = O[(uint64_t)b * nblk];
    e1 = (int)b + 1 < nb ? O[(uint64_t)(b + 1) * nblk] : O[last] + H[last];
}

// Closed-form source counts folded into the last batch's slice count
// (uniform degree): node v's edges [m0 + (v - n0) d, + d) overlap [lo, hi).
// Every bucket then gets at least one work item, so every node is visited.
struct SrcFold {
    uint64_t lo, hi, m0, n0, d;
    int on;
};
__device__ __forceinline__ uint64_t src_overlap(const SrcFold &f, uint64_t v) {
    if (v < f.n0) return 0u;
    const uint64_t a = f.m0 + (v - f.n0) * f.d, b = a + f.d;
    const uint64_t x = a > f.lo ? a : f.lo, y = b < f.hi ? b : f.hi;
    return y > x ? y - x : 0u;
}

// Owner-routed counts (multi-GPU full histogram): instead of a local n-word
// array summed by a collective afterwards, node v's counter lives on owner
// g = v / slice at ptr[g][v - g * slice] -- the owner's own memory or a peer
// mapping of it (NVLink) -- and every count CTA adds its bucket's counters
// there with red.add as soon as the bucket is counted: the reduce-scatter of
// the histograms (analytics.py:78-82, Consumer.merge) fused into the count
// kernel, its traffic overlapped with the counting of the other buckets.
// slice is a multiple of 2^16 >= kSliceMax, so one CTA's nodes have at most
// two owners.
constexpr int kMaxOwners = 16;
struct Route {
    uint32_t *ptr[kMaxOwners];
    uint32_t slice;  // nodes per owner
    int n;           // owners (0: local counts)
};

__global__ void __launch_bounds__(kHistThreads) count_plan_kernel(const uint32_t *__restrict__ O,
                                                                  const uint32_t *__restrict__ H, uint32_t nblk,
                                                                  int nb, uint32_t *__restrict__ items,
                                                                  uint32_t *__restrict__ n_items, int all_buckets) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nb; b0 += kHistThreads) {
        const uint32_t b = b0 + threadIdx.x;
        uint32_t chunks = 0;
        if ((int)b < nb) {
            uint32_t e0, e1;
            bucket_range(O, H, nblk, nb, b, e0, e1);
            chunks = e1 > e0 ? (e1 - e0 + kCountChunk - 1) / kCountChunk : (all_buckets ? 1u : 0u);
        }
        const uint32_t carry = carry_s;
        const uint32_t base = carry + block_exclusive_scan(chunks, warp_sums);
        for (uint32_t c = 0; c < chunks; ++c) items[base + c] = b | (c << kBucketBits);
        __syncthreads();  // every thread has read carry_s
        if (threadIdx.x == kHistThreads - 1) carry_s = base + chunks;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_items = carry_s;
}

// Step 3: CTA (item, s) counts the entries of one chunk of bucket b that fall
// in slice s (nodes (b << shift) + (s << kSliceLg) + [0, 2^kSliceLg)) and
// adds them to counts: plain read-modify-write when the chunk is the whole
// bucket (the CTA owns those counters), atomics when the bucket is split.
// The 2^spb_lg CTAs of an item are adjacent in the grid, so the chunk is
// read from HBM about once and from L2 by the others.  (A cluster variant
// that reads the chunk once and routes each entry to the owning CTA with a
// distributed-shared-memory red.add measured 3x slower.)
// OFF16: the entries are u16 offsets within one-slice buckets (spb_lg = 0).
// ROUTED: counts is unused, every non-zero counter (folded sources included)
// goes to its owner through `route` with one red.add.
template <typename CountT, bool OFF16 = false, bool ROUTED = false>
__global__ void __launch_bounds__(kHistThreads) slice_count_kernel(const uint32_t *__restrict__ sorted,
                                                                   const uint32_t *__restrict__ O,
                                                                   const uint32_t *__restrict__ H, uint32_t nblk,
                                                                   int nb, const uint32_t *__restrict__ items,
                                                                   const uint32_t *__restrict__ n_items, uint32_t n,
                                                                   uint32_t bw, int spb_lg,
                                                                   CountT *__restrict__ counts, SrcFold fold,
                                                                   Route route = Route{}) {
    extern __shared__ uint32_t c[];
    const uint32_t it = blockIdx.x >> spb_lg;
    if (it >= *n_items) return;
    const uint32_t item = items[it];
    const uint32_t b = item & ((1u << kBucketBits) - 1), chunk = item >> kBucketBits;
    PARBA_CHECK((int)b < nb);
    const uint32_t s = blockIdx.x & ((1u << spb_lg) - 1);
    for (uint32_t k = threadIdx.x; k < (spb_lg ? (uint32_t)kSliceNodes : bw); k += blockDim.x) c[k] = 0;
    __syncthreads();
    uint32_t e0, e1;
    bucket_range(O, H, nblk, nb, b, e0, e1);
    const bool split = e1 - e0 > kCountChunk;
    const uint32_t k0 = e0 + chunk * kCountChunk;
    const uint32_t k1 = e1 - k0 > kCountChunk ? k0 + kCountChunk : e1;
    const uint32_t smask = (1u << spb_lg) - 1;
    // bucket width bw: 2^(15 + spb_lg) (slices of 2^15 nodes) or, with
    // spb_lg = 0, any width up to kSliceMax held in one slice
    const uint32_t base_b = b * bw;
    const uint32_t imask = spb_lg ? (uint32_t)(kSliceNodes - 1) : 0xffffffffu;
    auto count = [&](uint32_t x) {
        const uint32_t l = x - base_b;
        if (((l >> kSliceLg) & smask) == s) atomicAdd(&c[l & imask], 1u);
    };
    auto count4 = [&](const uint4 &w) {
        count(w.x);
        count(w.y);
        count(w.z);
        count(w.w);
    };
    constexpr int NL = PARBA_COUNT_LOADS;
    const uint32_t bd = blockDim.x;
    if constexpr (OFF16) {
        // u16 offsets: scalar head to a 16-byte boundary, 8 entries per
        // 16-byte word, tail
        PARBA_CHECK(spb_lg == 0);
        const uint16_t *s16 = reinterpret_cast<const uint16_t *>(sorted);
        auto c2 = [&](uint32_t w) {
            atomicAdd(&c[w & 0xffffu], 1u);
            atomicAdd(&c[w >> 16], 1u);
        };
        const uint32_t h0 = ((k0 + 7u) & ~7u) < k1 ? ((k0 + 7u) & ~7u) : k1;
        if (k0 + threadIdx.x < h0) atomicAdd(&c[__ldg(s16 + k0 + threadIdx.x)], 1u);
        const uint32_t nv8 = (k1 - h0) / 8;
        const uint4 *w4 = reinterpret_cast<const uint4 *>(s16 + h0);
        uint32_t j = threadIdx.x;
        for (; j + (NL - 1) * bd < nv8; j += NL * bd) {
            uint4 w[NL];
#pragma unroll
            for (int u = 0; u < NL; ++u) w[u] = __ldg(w4 + j + u * bd);
#pragma unroll
            for (int u = 0; u < NL; ++u) {
                c2(w[u].x);
                c2(w[u].y);
                c2(w[u].z);
                c2(w[u].w);
            }
        }
        for (; j < nv8; j += bd) {
            const uint4 w = __ldg(w4 + j);
            c2(w.x);
            c2(w.y);
            c2(w.z);
            c2(w.w);
        }
        const uint32_t t8 = h0 + 8 * nv8;
        if (t8 + threadIdx.x < k1) atomicAdd(&c[__ldg(s16 + t8 + threadIdx.x)], 1u);
    } else {
    // scalar head to a 16-byte boundary, then 16-byte words with four loads in
    // flight per thread (the reads are latency-bound), tail
    const uint32_t a0 = ((k0 + 3u) & ~3u) < k1 ? ((k0 + 3u) & ~3u) : k1;
    if (k0 + threadIdx.x < a0) count(__ldg(sorted + k0 + threadIdx.x));
    const uint32_t nv = (k1 - a0) / 4;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(sorted + a0);
    uint32_t j = threadIdx.x;
    for (; j + (NL - 1) * bd < nv; j += NL * bd) {
        uint4 w[NL];
#pragma unroll
        for (int u = 0; u < NL; ++u) w[u] = __ldg(s4 + j + u * bd);
#pragma unroll
        for (int u = 0; u < NL; ++u) count4(w[u]);
    }
    for (; j < nv; j += bd) count4(__ldg(s4 + j));
    const uint32_t t0 = a0 + 4 * nv;
    if (t0 + threadIdx.x < k1) count(__ldg(sorted + t0 + threadIdx.x));
    }
    __syncthreads();
    const uint64_t v0 = (uint64_t)base_b + ((uint64_t)s << kSliceLg);
    const uint32_t sw = spb_lg ? (uint32_t)kSliceNodes : bw;
    if constexpr (ROUTED) {
        static_assert(sizeof(CountT) == 4, "routed counts are u32");
        // nodes [v0, v0 + lim) of this CTA: owner g0 below bnd, g0 + 1 from there
        const uint32_t lim = v0 >= n ? 0u : (uint64_t)sw < n - v0 ? sw : (uint32_t)(n - v0);
        const bool addsrc = fold.on && (!split || chunk == 0);
        const uint32_t g0 = (uint32_t)(v0 / route.slice);
        const uint64_t bnd = (uint64_t)(g0 + 1) * route.slice;
        PARBA_CHECK(lim == 0 || (int)g0 < route.n);
        uint32_t *const p0 = route.ptr[g0];
        uint32_t *const p1 = (int)g0 + 1 < route.n ? route.ptr[g0 + 1] : nullptr;
        const uint32_t o0 = (uint32_t)(v0 - (uint64_t)g0 * route.slice);
        for (uint32_t k = threadIdx.x; k < lim; k += blockDim.x) {
            const uint64_t v = v0 + k;
            const uint32_t x = c[k] + (addsrc ? (uint32_t)src_overlap(fold, v) : 0u);
            if (x) atomicAdd(v < bnd ? p0 + o0 + k : p1 + (v - bnd), x);  // RED.ADD (local or peer)
        }
        return;
    }
    if (split) {  // the bucket's first chunk also adds the folded sources
        const bool addsrc = fold.on && chunk == 0;
        for (uint32_t k = threadIdx.x; k < sw; k += blockDim.x) {
            const uint64_t v = v0 + k;
            const uint64_t x = c[k] + (addsrc && v < n ? src_overlap(fold, v) : 0u);
            if (v < n && x) atomicAdd(counts + v, (CountT)x);
        }
        return;
    }
    // the CTA owns these counters: read-modify-write, PARBA_FLUSH_UNROLL
    // independent loads in flight per thread (one round trip per group
    // instead of one per counter)
    const uint32_t lim = v0 >= n ? 0u : (uint64_t)sw < n - v0 ? sw : (uint32_t)(n - v0);
    constexpr int U = PARBA_FLUSH_UNROLL;
    uint32_t k = threadIdx.x;
    if (fold.on) {
        for (; k + (U - 1) * blockDim.x < lim; k += U * blockDim.x) {
            CountT old[U];
#pragma unroll
            for (int u = 0; u < U; ++u) old[u] = counts[v0 + k + u * blockDim.x];
#pragma unroll
            for (int u = 0; u < U; ++u)
                counts[v0 + k + u * blockDim.x] =
                    old[u] + c[k + u * blockDim.x] + (CountT)src_overlap(fold, v0 + k + u * blockDim.x);
        }
        for (; k < lim; k += blockDim.x) counts[v0 + k] += c[k] + (CountT)src_overlap(fold, v0 + k);
        return;
    }
    for (; k + (U - 1) * blockDim.x < lim; k += U * blockDim.x) {
        CountT old[U];
#pragma unroll
        for (int u = 0; u < U; ++u) old[u] = counts[v0 + k + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < U; ++u) counts[v0 + k + u * blockDim.x] = old[u] + c[k + u * blockDim.x];
    }
    for (; k < lim; k += blockDim.x) counts[v0 + k] += c[k];
}

// Step 3 for positions (degree sequences): like slice_count_kernel over the
// position domain, then each slice's position counts are summed per owning
// node (dense owner map, read in order; owners are non-decreasing in the
// position, so a warp reduces runs of equal owners with shuffles) and the
// run totals are added to counts with atomics (a node's positions may span
// slices).  Positions >= m are never stored; positions < m0 never occur.
template <typename CountT>
__global__ void __launch_bounds__(kHistThreads) slice_count_pos_kernel(
    const uint32_t *__restrict__ sorted, const uint32_t *__restrict__ O, const uint32_t *__restrict__ H,
    uint32_t nblk, int nb, const uint32_t *__restrict__ items, const uint32_t *__restrict__ n_items, uint64_t m0,
    uint64_t m, int shift, int spb_lg, const uint32_t *__restrict__ dense, CountT *__restrict__ counts) {
    extern __shared__ uint32_t c[];
    const uint32_t it = blockIdx.x >> spb_lg;
    if (it >= *n_items) return;
    const uint32_t item = items[it];
    const uint32_t b = item & ((1u << kBucketBits) - 1), chunk = item >> kBucketBits;
    const uint32_t s = blockIdx.x & ((1u << spb_lg) - 1);
    for (int k = threadIdx.x; k < kSliceNodes; k += blockDim.x) c[k] = 0;
    __syncthreads();
    uint32_t e0, e1;
    bucket_range(O, H, nblk, nb, b, e0, e1);
    const uint32_t k0 = e0 + chunk * kCountChunk;
    const uint32_t k1 = e1 - k0 > kCountChunk ? k0 + kCountChunk : e1;
    const uint32_t smask = (1u << spb_lg) - 1;
    for (uint32_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const uint32_t x = __ldg(sorted + k);
        if (((x >> kSliceLg) & smask) == s) atomicAdd(&c[x & (kSliceNodes - 1)], 1u);
    }
    __syncthreads();
    const uint64_t p0 = ((uint64_t)b << shift) + ((uint64_t)s << kSliceLg);
    const int lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < kSliceNodes; k += blockDim.x) {  // warp-uniform trip count
        const uint64_t pos = p0 + k;
        const bool in = pos >= m0 && pos < m;
        uint32_t x = in ? c[k] : 0u;
        const uint32_t v = in ? __ldg(dense + (pos - m0)) : 0xffffffffu;
        // inclusive segmented sum over lanes with the same owner (runs)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            const uint32_t w = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o && w == v) x += y;
        }
        const uint32_t vn = __shfl_down_sync(0xffffffffu, v, 1);
        if (in && x && (lane == 31 || vn != v)) atomicAdd(counts + v, (CountT)x);
    }
}

}  // namespace parba
