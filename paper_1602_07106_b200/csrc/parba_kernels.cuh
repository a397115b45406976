// parba_kernels.cuh -- sm_100a kernels of the Sanders-Schulz edge generator.
//
// The hot path is generateEdge(i) (generator.py:172-181;
// _kernels.py:63-75): r := 2i+1; repeat r := h(r) until r is even (or falls
// into the seed region); emit (src(i), tgt(r)).  Chain lengths are geometric
// (mean 2), so one-edge-per-lane code would idle ~2/3 of every warp.  The
// engine here is warp-centric:
//
//   phase 1  every lane takes the first probe of 8 edges of a 256-edge,
//            256-aligned warp tile.  r0 = 2i+1 = 2B + (2j+1), so by CRC
//            linearity crc(0,r0) = crc(0,2B) ^ crc(0,2j+1): a warp-uniform
//            value per tile XOR a per-lane register constant -- the first
//            probe (half of all probes) needs no table lookup.  About half
//            the edges finish here; the rest go to a per-warp smem queue.
//   phase 2  lanes pop queued chains (ballot/popc refill) and probe until
//            the queue is empty; chains still running stay in registers and
//            carry over into the next tile, so lanes never wait for the
//            longest chain of a tile.
//   sink     Store: targets land in a 2-deep smem ring of tile buffers; a
//            tile is written out (16-byte streaming stores, fully coalesced)
//            once its last chain finished.  Window/Full: a finished chain
//            increments its target's counter directly (E never stored).
//
// Persistent grid: one resident wave of CTAs, warps stride over tiles.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "parba_device.cuh"

namespace parba {

constexpr int kTile = 256;                 // edges per warp tile (power of two)
constexpr int kEpl = kTile / 32;           // edges per lane in phase 1
constexpr int kWarps = 8;                  // warps per CTA
constexpr int kThreads = kWarps * 32;

enum SinkKind { kStore = 0, kWindow = 1, kFull = 2 };
constexpr int kTabBytes = (sizeof(CrcTables) + 15) / 16 * 16;

struct StoreArgs {
    uint64_t *out;                         // 2*(hi-lo) u64, 16-byte aligned
    unsigned long long *win;               // window counts (K)
    uint32_t *full;                        // full counts (n)
};

template <int SINK>
struct WarpSmem;

template <>
struct WarpSmem<kStore> {
    uint64_t stage[2][kTile];  // targets of the two tiles in flight
    uint64_t qr[kTile];        // pending chain values
    uint16_t qs[kTile];        // pending slots: buf*kTile + j
};
template <>
struct WarpSmem<kWindow> {
    uint64_t qr[kTile];
};
template <>
struct WarpSmem<kFull> {
    uint64_t qr[kTile];
};

template <int SINK>
constexpr size_t tile_smem_bytes() { return kTabBytes + kWarps * sizeof(WarpSmem<SINK>); }

template <int SINK>
__device__ __forceinline__ void finish(WarpSmem<SINK> &w, uint32_t slot, uint64_t r,
                                       const DevParams &p, const StoreArgs &a) {
    if constexpr (SINK == kStore) {
        (&w.stage[0][0])[slot] = target_of(r, p);  // slot spans both ring buffers
    } else if constexpr (SINK == kWindow) {
        // target < K  <=>  (r>>1) < win_lim for generated positions
        if (r >= p.stop) {
            if ((r >> 1) < p.win_lim) atomicAdd(a.win + target_of(r, p), 1ull);
        } else {
            uint64_t t = __ldg(p.seed + r);
            if (t < p.K) atomicAdd(a.win + t, 1ull);
        }
    } else {
        atomicAdd(a.full + target_of(r, p), 1u);
    }
}

template <class Hash, int NCH, int SINK>
__global__ void __launch_bounds__(kThreads, 3)
tile_kernel(DevParams p, uint64_t lo, uint64_t hi, uint64_t tile0, uint64_t ntiles,
            StoreArgs a, unsigned long long *probes_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CrcTables &tabs = *reinterpret_cast<CrcTables *>(smem_raw);
    WarpSmem<SINK> *wsm = reinterpret_cast<WarpSmem<SINK> *>(smem_raw + kTabBytes);
    build_crc_tables(tabs);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem<SINK> &w = wsm[wib];
    const unsigned ltmask = lanemask_lt();
    const uint64_t gw = (uint64_t)blockIdx.x * kWarps + wib;
    const uint64_t nw = (uint64_t)gridDim.x * kWarps;

    // crc(0, 2j+1) for this lane's phase-1 edges j = lane + 32k (2j+1 < 512).
    uint32_t clow[kEpl];
#pragma unroll
    for (int k = 0; k < kEpl; ++k) clow[k] = crc0<2>(tabs, 2u * (lane + 32u * k) + 1u);

    bool act = false;        // lane holds a running chain
    uint64_t r = 0;
    uint32_t slot = 0;
    uint32_t head = 0, tail = 0;  // queue cursors (warp-uniform)
    unsigned long long probes = 0;
    uint64_t prev_base = 0;
    bool have_prev = false;
    uint32_t buf = 0;

    // Write a finished tile out of buffer b (store mode).
    auto flush = [&](uint32_t b, uint64_t base) {
        if constexpr (SINK == kStore) {
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kEpl; ++k) {
                const uint32_t j = lane + 32u * k;
                const uint64_t i = base + j;
                if (i >= lo && i < hi) {
                    ulonglong2 v = make_ulonglong2(source_of(i, p), w.stage[b][j]);
                    __stcs(reinterpret_cast<ulonglong2 *>(a.out + 2 * (i - lo)), v);
                }
            }
            __syncwarp();
        }
    };

    // One probe on every active lane; finished chains go to the sink.
    auto step = [&]() {
        if (act) {
            r = Hash::probe(tabs, r, p);
            ++probes;
            if (r < p.stop || (r & 1ull) == 0) {
                finish<SINK>(w, slot, r, p, a);
                act = false;
            }
        }
    };

    for (uint64_t t = gw; t < ntiles; t += nw) {
        const uint64_t base = (tile0 + t) * kTile;
        // ---- phase 1: first probe of all edges of the tile
        uint32_t cb = 0;
        if constexpr (Hash::kHasCrc) cb = crc0<NCH>(tabs, 2 * base);
#pragma unroll
        for (int k = 0; k < kEpl; ++k) {
            const uint32_t j = lane + 32u * k;
            const uint64_t i = base + j;
            const bool valid = (i >= lo) && (i < hi);
            const uint64_t r0 = 2 * i + 1;
            uint64_t r1;
            if constexpr (Hash::kHasCrc) r1 = Hash::from_crc(cb ^ clow[k], r0, p);
            else r1 = Hash::probe(tabs, r0, p);
            const bool done = (r1 < p.stop) || ((r1 & 1ull) == 0);
            if (valid) {
                ++probes;
                if (done) finish<SINK>(w, buf * kTile + j, r1, p, a);
            }
            const bool pend = valid && !done;
            const unsigned m = __ballot_sync(0xffffffffu, pend);
            if (pend) {
                const uint32_t pos = (tail + __popc(m & ltmask)) & (kTile - 1);
                w.qr[pos] = r1;
                if constexpr (SINK == kStore) w.qs[pos] = (uint16_t)(buf * kTile + j);
            }
            tail += __popc(m);
        }
        __syncwarp();
        // ---- phase 2: drain the queue with lane refill
        while (tail != head) {
            const unsigned idle = __ballot_sync(0xffffffffu, !act);
            const uint32_t avail = tail - head;
            if (!act) {
                const uint32_t rank = __popc(idle & ltmask);
                if (rank < avail) {
                    const uint32_t pos = (head + rank) & (kTile - 1);
                    r = w.qr[pos];
                    if constexpr (SINK == kStore) slot = w.qs[pos];
                    act = true;
                }
            }
            const uint32_t took = min((uint32_t)__popc(idle), avail);
            head += took;
            step();
        }
        // ---- store: flush the previous tile once none of its chains runs
        if constexpr (SINK == kStore) {
            if (have_prev) {
                const uint32_t pb = buf ^ 1u;
                while (__any_sync(0xffffffffu, act && (slot / kTile) == pb)) step();
                flush(pb, prev_base);
            }
            prev_base = base;
            have_prev = true;
            buf ^= 1u;
        }
    }
    // ---- drain the chains still running, then flush the last tile
    while (__any_sync(0xffffffffu, act)) step();
    if constexpr (SINK == kStore) {
        if (have_prev) flush(buf ^ 1u, prev_base);
    }
    // ---- probes: warp reduce, one atomic per warp
    if (probes_out) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) probes += __shfl_xor_sync(0xffffffffu, probes, o);
        if (lane == 0) atomicAdd(probes_out, probes);
    }
}

// ---------------------------------------------------------------------------
// Generic kernels (not the bench path): arbitrary chain starts / ID lists.

template <class Hash, int NCH>
__global__ void __launch_bounds__(256)
chains_kernel(DevParams p, const uint64_t *__restrict__ r0, uint64_t count, uint64_t stop,
              uint64_t *__restrict__ out, const uint64_t *__restrict__ ids,
              uint64_t *__restrict__ pairs, unsigned long long *probes_out) {
    __shared__ CrcTables tabs;
    build_crc_tables(tabs);
    __syncthreads();
    unsigned long long probes = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = ids ? 2 * ids[k] + 1 : r0[k];
        do {  // body at least once (generator.py:146-154)
            r = Hash::probe(tabs, r, p);
            ++probes;
        } while (!(r < stop || (r & 1ull) == 0));
        if (ids) {
            reinterpret_cast<ulonglong2 *>(pairs)[k] = make_ulonglong2(source_of(ids[k], p), target_of(r, p));
        } else {
            out[k] = r;
        }
    }
    if (probes_out) {
        for (int o = 16; o > 0; o >>= 1) probes += __shfl_xor_sync(0xffffffffu, probes, o);
        if ((threadIdx.x & 31) == 0 && probes) atomicAdd(probes_out, probes);
    }
}

template <class Hash, int NCH>
__global__ void __launch_bounds__(256)
hash_kernel(DevParams p, const uint64_t *__restrict__ r, uint64_t count, uint64_t *__restrict__ out) {
    __shared__ CrcTables tabs;
    build_crc_tables(tabs);
    __syncthreads();
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = Hash::probe(tabs, r[k], p);
}

// Source endpoints of a window/full count in closed form: node v owns edges
// [m0+(v-n0)d, m0+(v-n0+1)d); its count grows by the overlap with [lo,hi).
template <typename CountT>
__global__ void source_counts_kernel(DevParams p, uint64_t lo, uint64_t hi, uint64_t vlo,
                                     uint64_t vhi, CountT *counts) {
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = p.m0 + (v - p.n0) * p.d, b = a + p.d;
        const uint64_t x = a > lo ? a : lo, y = b < hi ? b : hi;
        if (y > x) counts[v] += (CountT)(y - x);
    }
}

}  // namespace parba

namespace parba {

// count_block on device (analytics.py:44-48): counts[id] += 1 for id < K.
__global__ void count_ids_kernel(const uint64_t *__restrict__ ids, uint64_t count, uint64_t K,
                                 unsigned long long *counts) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = ids[k];
        if (v < K) atomicAdd(counts + v, 1ull);
    }
}

}  // namespace parba
