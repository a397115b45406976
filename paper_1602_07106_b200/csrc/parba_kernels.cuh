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
//            value per tile XOR a constant read from a 1 KB smem table
//            (conflict-free, lane-consecutive) -- the first probe (half of
//            all probes) needs one lookup instead of NB.  About half
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
// Template axes: Hash (CRC with NB table bytes / SIMPLE; narrow = every chain
// value < 2^32), SINK, SEED (m0 > 0 or n0 > 0: offsets and the seed stop).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "parba_device.cuh"

namespace parba {

constexpr int kTile = 256;                 // edges per warp tile (power of two)
constexpr int kQueue = 512;                // per-warp pending ring (>= kTile + 31)
constexpr int kEpl = kTile / 32;           // edges per lane in phase 1
#ifndef PARBA_WARPS
#define PARBA_WARPS 32
#endif
#ifndef PARBA_MINB_STORE
#define PARBA_MINB_STORE 1
#endif
#ifndef PARBA_MINB_STREAM
#define PARBA_MINB_STREAM 1
#endif
constexpr int kWarps = PARBA_WARPS;        // warps per CTA
constexpr int kThreads = kWarps * 32;

enum SinkKind { kStore = 0, kWindow = 1, kFull = 2 };

struct SinkArgs {
    uint64_t *out;                         // store: 2*(hi-lo) u64, 16-byte aligned
    unsigned long long *win;               // window counts (K)
    uint32_t *full;                        // full counts (n)
};

// Per-warp shared state.  R = chain value type (u32 in narrow mode).
// Store queue entries pack the chain value and its stage slot (9 bits) into
// one u64 -- value in the low 55 bits -- when every position is < 2^52
// (Hash::kPack); otherwise the slot goes to a separate u16 ring.
template <int SINK, class R>
struct WarpSmem {
    uint64_t qe[kQueue];       // pending (slot << 55) | value   (ring)
    uint16_t qs[kQueue];       // pending slots when !kPack
    R stage[2][kTile];         // terminal chain values of the two tiles in flight
};
template <class R>
struct WarpSmem<kWindow, R> {
    R qr[kQueue];
};
template <class R>
struct WarpSmem<kFull, R> {
    R qr[kQueue];
};

// Dynamic shared memory: [CRC tables][crc(0,2j+1) table][per-warp state].
template <class Hash>
constexpr size_t tile_smem_fixed() {
    return Hash::kHasCrc ? (Hash::kTableWords + kTile) * 4 : 0;
}
template <class Hash, int SINK>
constexpr size_t tile_smem_per_warp() {
    return sizeof(WarpSmem<SINK, typename Hash::R>);
}
constexpr uint64_t kValueMask = (1ull << 55) - 1;

// A chain finished with terminal value r: hand its target to the sink.
template <bool NARROW, bool SEED, int SINK, class R>
__device__ __forceinline__ void finish(uint32_t stage_s, uint32_t slot, uint64_t r, const DevParams &p,
                                       const SinkArgs &a) {
    if constexpr (SINK == kStore) {
        sts_t<R>(stage_s + slot * (uint32_t)sizeof(R), (R)r);  // target computed at flush, all lanes busy
    } else if constexpr (SINK == kWindow) {
        if (SEED && r < p.stop) {
            const uint64_t t = __ldg(p.seed + r);
            if (t < p.K) atomicAdd(a.win + t, 1ull);
        } else if (NARROW ? ((uint32_t)r < p.win_rlim32) : (r < p.win_rlim)) {
            // generated target < K  <=>  r < win_rlim
            atomicAdd(a.win + source_of<NARROW, SEED>(r >> 1, p), 1ull);
        }
    } else {
        atomicAdd(a.full + target_of<NARROW, SEED>(r, p), 1u);
    }
}

template <class Hash, int SINK, bool SEED>
__global__ void __launch_bounds__(kThreads, SINK == kStore ? PARBA_MINB_STORE : PARBA_MINB_STREAM)
tile_kernel(DevParams p, uint64_t lo, uint64_t hi, uint64_t tile0, uint64_t ntiles,
            SinkArgs a, unsigned long long *probes_out) {
    using R = typename Hash::R;
    constexpr bool NARROW = Hash::kNarrow;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *tabs_p = reinterpret_cast<uint32_t *>(smem_raw);
    uint32_t *clow_s = tabs_p + Hash::kTableWords;  // crc(0, 2j+1), j < kTile (2j+1 < 512)
    const uint32_t tabs = opaque(smem_addr(tabs_p));
    WarpSmem<SINK, R> *wsm = reinterpret_cast<WarpSmem<SINK, R> *>(
        smem_raw + (Hash::kHasCrc ? (Hash::kTableWords + kTile) * 4 : 0));
    if constexpr (Hash::kHasCrc) {
        Hash::build(tabs_p, p.k0);
        for (int j = threadIdx.x; j < kTile; j += blockDim.x)
            clow_s[j] = crc32c_u64_bitwise(0u, 2u * (uint32_t)j + 1u);
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;  // warps per CTA (<= kWarps; fewer when smem is tight)
    WarpSmem<SINK, R> &w = wsm[wib];
    // shared-window addresses of this warp's queue and stage (kept in registers)
    uint32_t qe_s, qs_s = 0, stage_s = 0;
    if constexpr (SINK == kStore) {
        qe_s = opaque(smem_addr(&w.qe[0]));
        qs_s = opaque(smem_addr(&w.qs[0]));
        stage_s = opaque(smem_addr(&w.stage[0][0]));
    } else {
        qe_s = opaque(smem_addr(&w.qr[0]));
    }
    const unsigned ltmask = lanemask_lt();
    const uint64_t gw = (uint64_t)blockIdx.x * wpc + wib;
    const uint64_t nw = (uint64_t)gridDim.x * wpc;

    uint32_t act = 0;             // 1: lane holds a running chain
    R r = 0;
    uint32_t slot = 0;
    uint32_t head = 0, tail = 0;  // queue cursors (warp-uniform)
    uint32_t tile_q0 = 0;         // queue cursor at the start of the current tile
    uint32_t probes = 0;          // per lane (< 2^32 per launch and lane)
    uint64_t prev_base = 0;
    bool have_prev = false;
    uint32_t buf = 0;

    auto is_done = [&](R v) -> bool {
        if constexpr (SEED) return ((uint32_t)v & 1u) == 0 || (uint64_t)v < p.stop;
        else return ((uint32_t)v & 1u) == 0;
    };

    // Write a finished tile out of buffer b (store mode): (source, target)
    // pairs from the staged terminal values, 16-byte streaming stores.
    // Interior tiles (all but the range ends) skip the per-edge bounds test.
    auto flush_t = [&](auto full_c, uint32_t b, uint64_t base) {
        [[maybe_unused]] constexpr bool FULL = decltype(full_c)::value;
        if constexpr (SINK == kStore) {
            ulonglong2 *o = reinterpret_cast<ulonglong2 *>(a.out) + (int64_t)(base - lo);
#pragma unroll
            for (int k = 0; k < kEpl; ++k) {
                const uint32_t j = lane + 32u * k;
                const uint64_t i = base + j;
                if (FULL || (i >= lo && i < hi)) {
                    const uint64_t tgt = target_of<NARROW, SEED, Hash::kR31>(
                        (uint64_t)lds_t<R>(stage_s + (b * kTile + j) * (uint32_t)sizeof(R)), p);
                    __stcs(o + j, make_ulonglong2(source_of<NARROW, SEED>(i, p), tgt));
                }
            }
        }
    };
    auto flush = [&](uint32_t b, uint64_t base) {
        if constexpr (SINK == kStore) {
            __syncwarp();
            if (base >= lo && base + kTile <= hi) flush_t(std::true_type{}, b, base);
            else flush_t(std::false_type{}, b, base);
            __syncwarp();
        }
    };

    // One probe on every lane (idle lanes hash a harmless stale value and
    // discard it: no divergent branch around the probe); finished chains go
    // to the sink.
    auto step = [&]() {
        const R nr = Hash::probe(tabs, r, p);
        probes += (uint32_t)act;
        uint32_t cont = (uint32_t)nr & 1u;  // odd: the chain continues
        if constexpr (SEED) cont &= (uint64_t)nr >= p.stop ? 1u : 0u;
        const uint32_t fin = act & (cont ^ 1u);
        act &= cont;
        r = nr;
        if (fin) finish<NARROW, SEED, SINK, R>(stage_s, slot, (uint64_t)nr, p, a);
    };

    // Pop queued chains into idle lanes.  FULLQ: at least 32 entries queued,
    // so every idle lane takes one (no availability test).
    auto refill = [&](auto fullq_c) {
        constexpr bool FULLQ = decltype(fullq_c)::value;
        const unsigned idle = ballot_all(!act);
        const uint32_t rank = __popc(idle & ltmask);
        const uint32_t avail = tail - head;
        if (!act && (FULLQ || rank < avail)) {
            const uint32_t pos = (head + rank) & (kQueue - 1);
            if constexpr (SINK == kStore) {
                const uint64_t e = lds_u64(qe_s + pos * 8);
                if constexpr (Hash::kPack) {
                    r = (R)(e & kValueMask);
                    slot = (uint32_t)(e >> 55);
                } else {
                    r = (R)e;
                    slot = lds_u16(qs_s + pos * 2);
                }
            } else {
                r = lds_t<R>(qe_s + pos * (uint32_t)sizeof(R));
            }
            act = 1;
        }
        if constexpr (FULLQ) head += (uint32_t)__popc(idle);
        else head += min((uint32_t)__popc(idle), avail);
    };

    // First probe of every edge of a tile (FULL: interior tile, no bounds test).
    auto phase1 = [&](auto full_c, uint64_t base, uint32_t cb) {
        constexpr bool FULL = decltype(full_c)::value;
#pragma unroll
        for (int k = 0; k < kEpl; ++k) {
            const uint32_t j = lane + 32u * k;
            const uint64_t i = base + j;
            const bool valid = FULL || ((i >= lo) && (i < hi));
            const R r0 = (R)(2 * base) + (R)(2 * j + 1);
            R r1;
            if constexpr (Hash::kHasCrc) r1 = Hash::from_crc(cb ^ clow_s[j], r0, p);
            else r1 = Hash::probe(tabs, r0, p);
            const bool done = is_done(r1);
            if constexpr (SINK == kStore)  // final unless pending
                sts_t<R>(stage_s + (buf * kTile + j) * (uint32_t)sizeof(R), r1);
            if constexpr (SINK != kStore) if (valid && done) finish<NARROW, SEED, SINK, R>(stage_s, buf * kTile + j, (uint64_t)r1, p, a);
            const bool pend = valid && !done;
            const unsigned m = ballot_all(pend);
            const uint32_t pos = (tail + __popc(m & ltmask)) & (kQueue - 1);
            if constexpr (SINK == kStore) {
                if constexpr (Hash::kPack) {
                    // predicated store, no branch: (slot << 55) | value
                    const uint32_t slot_hi = ((buf * kTile + j) << 23);
                    sts_u64_if(pend, qe_s + pos * 8, ((uint64_t)slot_hi << 32) | (uint64_t)r1);
                } else if (pend) {
                    sts_u64(qe_s + pos * 8, (uint64_t)r1);
                    sts_u16(qs_s + pos * 2, (uint16_t)(buf * kTile + j));
                }
            } else {
                sts_t_if<R>(pend, qe_s + pos * (uint32_t)sizeof(R), r1);
            }
            tail += __popc(m);
            probes += valid ? 1u : 0u;
        }
    };

    for (uint64_t t = gw; t < ntiles; t += nw) {
        const uint64_t base = (tile0 + t) * kTile;
        // ---- phase 1: first probe of all edges of the tile
        tile_q0 = tail;  // queue position where this tile's entries start
        uint32_t cb = 0;
        if constexpr (Hash::kHasCrc) cb = Hash::crc(tabs, 2 * base, p);
        if (base >= lo && base + kTile <= hi) phase1(std::true_type{}, base, cb);
        else phase1(std::false_type{}, base, cb);
        __syncwarp();
        // ---- phase 2: pop queued chains into idle lanes and probe while at
        // least a full warp of entries is queued (the < 32 newest entries
        // carry over to the next tile, so every refill can fill every idle lane)
        while (tail - head >= 32u) {
            refill(std::true_type{});
            step();
        }
        // ---- store: flush the previous tile once none of its chains runs
        if constexpr (SINK == kStore) {
            if (have_prev) {
                const uint32_t pb = buf ^ 1u;
                // entries of the previous tile still queued (only when this
                // tile pushed fewer than 32): pop them first
                while ((int32_t)(tile_q0 - head) > 0) {
                    refill(std::false_type{});
                    step();
                }
                while (__any_sync(0xffffffffu, act && (slot / kTile) == pb)) step();
                flush(pb, prev_base);
            }
            prev_base = base;
            have_prev = true;
            buf ^= 1u;
        }
    }
    // ---- drain the queue and the chains still running, then flush the last tile
    while (tail != head) {
        refill(std::false_type{});
        step();
    }
    while (__any_sync(0xffffffffu, act)) step();
    if constexpr (SINK == kStore) {
        if (have_prev) flush(buf ^ 1u, prev_base);
    }
    // ---- probes: warp reduce, one atomic per warp
    if (probes_out) {
        unsigned long long pr = probes;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
        if (lane == 0) atomicAdd(probes_out, pr);
    }
}

// ---------------------------------------------------------------------------
// Generic kernels (not the bench path): arbitrary chain starts / ID lists,
// full 64-bit values.

template <class Hash>
__global__ void __launch_bounds__(256)
chains_kernel(DevParams p, const uint64_t *__restrict__ r0, uint64_t count, uint64_t stop,
              uint64_t *__restrict__ out, const uint64_t *__restrict__ ids,
              uint64_t *__restrict__ pairs, unsigned long long *probes_out) {
    __shared__ uint32_t tabs_p[Hash::kTableWords > 0 ? Hash::kTableWords : 1];
    Hash::build(tabs_p, p.k0);
    __syncthreads();
    const uint32_t tabs = opaque(smem_addr(tabs_p));
    unsigned long long probes = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = ids ? 2 * ids[k] + 1 : r0[k];
        do {  // body at least once (generator.py:146-154)
            r = Hash::probe(tabs, r, p);
            ++probes;
        } while (!(r < stop || (r & 1ull) == 0));
        if (ids) {
            reinterpret_cast<ulonglong2 *>(pairs)[k] =
                make_ulonglong2(source_of<false, true>(ids[k], p), target_of<false, true>(r, p));
        } else {
            out[k] = r;
        }
    }
    if (probes_out) {
        for (int o = 16; o > 0; o >>= 1) probes += __shfl_xor_sync(0xffffffffu, probes, o);
        if ((threadIdx.x & 31) == 0 && probes) atomicAdd(probes_out, probes);
    }
}

template <class Hash>
__global__ void __launch_bounds__(256)
hash_kernel(DevParams p, const uint64_t *__restrict__ r, uint64_t count, uint64_t *__restrict__ out) {
    __shared__ uint32_t tabs_p[Hash::kTableWords > 0 ? Hash::kTableWords : 1];
    Hash::build(tabs_p, p.k0);
    __syncthreads();
    const uint32_t tabs = opaque(smem_addr(tabs_p));
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
