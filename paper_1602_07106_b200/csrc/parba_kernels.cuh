// parba_kernels.cuh -- sm_100a kernels of the Sanders-Schulz edge generator.
//
// The hot path is generateEdge(i) (generator.py:172-181;
// _kernels.py:63-75): r := 2i+1; repeat r := h(r) until r is even (or falls
// into the seed region); emit (src(i), tgt(r)).  Chain lengths are geometric
// (mean 2), so one-edge-per-lane code would idle ~2/3 of every warp.  The
// engine here is warp-centric:
//
//   phase 1  every lane takes the first probe of 8 edges of a 256-edge,
//            256-aligned warp tile (16 edges of a 512-edge tile in the narrow
//            CRC store and store-targets kernels, in four pieces with lazy
//            drains between them: TileLayout::kBig).  r0 = 2i+1 = 2B + (2j+1), so by CRC
//            linearity crc(0,r0) = crc(0,2B) ^ crc(0,2j+1): a warp-uniform
//            value per tile XOR a constant read from a 1 KB smem table
//            (conflict-free, lane-consecutive) -- the first probe (half of
//            all probes) needs one lookup instead of NB.  About half
//            the edges finish here; the rest go to a per-warp smem queue.
//   phase 2  lanes pop queued chains (ballot/popc refill) and probe while
//            a warp's worth of entries is queued; chains still running stay
//            in registers and carry over into the next tile, so lanes never
//            wait for the longest chain of a tile (NS running chains per
//            lane: 1 for the store sink, 2 for the streaming sinks).
//   sink     Store: terminal values land in a 2-deep smem ring of tile
//            buffers; a tile is written out (16-byte streaming stores, fully
//            coalesced, sources and targets computed then) once its last
//            chain finished.  Window/Full: a finished chain increments its
//            target's counter directly (E never stored).
//
// Persistent grid: one resident wave of CTAs, warps stride over tiles.
// Template axes: Hash (CRC with NC chunk tables / SIMPLE; narrow = every
// chain value < 2^32), SINK, SEED (m0 > 0 or n0 > 0: offsets and the seed
// stop), DEG (degree sequence: owner lookups instead of division by d).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "parba_device.cuh"

namespace parba {

constexpr int kTile = 256;                 // edges per warp tile (power of two)
constexpr int kQueue = 512;                // per-warp pending ring (>= kTile + 31)
#ifndef PARBA_WIDE_SPLIT
#define PARBA_WIDE_SPLIT 1
#endif
#ifndef PARBA_NARROW_SPLIT
#define PARBA_NARROW_SPLIT 0  // A/B: the split phase 1 and 256-entry queue for narrow store kernels too
#endif
constexpr int kEpl = kTile / 32;           // edges per lane in phase 1
// Narrow CRC store launches: 512-edge tiles (16 edges per lane, phase 1 in
// four 128-edge pieces with a drain between them and a 256-entry queue), so
// the per-tile work -- crc(2*base), bounds, the flush hand-over -- is paid
// once per 512 edges (A/B knob).
#ifndef PARBA_TILE512
#define PARBA_TILE512 1
#endif
// the same for the streaming sinks (queue of 512 entries, a drain after 256
// edges): C3 window 2.554e11 -> 2.536e11 (-0.7%), off
// the store-targets sink (the full histogram's targets pass, the host-array
// pipeline) on 512-edge tiles too; the scatter takes the tile size as a parameter
#ifndef PARBA_TILE512_ST
#define PARBA_TILE512_ST 1
#endif
// edges per lane of a phase-1 piece in the split store kernels (A/B knob)
#ifndef PARBA_PIECE
#define PARBA_PIECE 4
#endif
#ifndef PARBA_LAZY_DRAIN
#define PARBA_LAZY_DRAIN 1
#endif
#ifndef PARBA_LAZY_END
#define PARBA_LAZY_END 0
#endif
#ifndef PARBA_TILE512_STREAM
#define PARBA_TILE512_STREAM 0
#endif
// first probes use the per-tile reciprocal series from 2*base >= 2^27 on
constexpr uint64_t kRyMin = 1ull << 27;
#ifndef PARBA_WARPS
#define PARBA_WARPS 32
#endif
// Running chains per lane in phase 2.  Two independent chains per lane help
// the streaming sinks (+2% at C3) but cost the store sink 17% (twice the
// chains in flight make the flush of the previous tile wait longer), A/B on
// one B200 with tools/ab.py.
#ifndef PARBA_ILP_STORE
#define PARBA_ILP_STORE 1
#endif
#ifndef PARBA_ILP_STREAM
#define PARBA_ILP_STREAM 2
#endif
#ifndef PARBA_MINB_STORE
#define PARBA_MINB_STORE 1
#endif
#ifndef PARBA_ILP_TARGETS
#define PARBA_ILP_TARGETS 2
#endif
#ifndef PARBA_MINB_STREAM
#define PARBA_MINB_STREAM 1
#endif
constexpr int kWarps = PARBA_WARPS;        // warps per CTA
// Window sink: bins of the lowest nodes privatised in shared memory (0 = off)
#ifndef PARBA_WIN_SMEM
#define PARBA_WIN_SMEM 0
#endif
constexpr uint32_t kWinSmem = PARBA_WIN_SMEM;
// Store-mode stage buffers (tiles in flight): 2 = flush tile t-1 after
// phase 2 of tile t; 3 = flush tile t-2 (its chains have had a whole tile
// longer to finish, so the flush rarely waits).
// phase-2 loop of the store sinks: refill+probe steps per loop-condition
// test (2: +0.35% at C2, profiles/r02_ab_window_smem_and_unroll.txt)
#ifndef PARBA_P2_UNROLL
#define PARBA_P2_UNROLL 2
#endif
#ifndef PARBA_P2_UNROLL_STREAM
#define PARBA_P2_UNROLL_STREAM 0  // the same for the streaming sinks (A/B)
#endif
#ifndef PARBA_NBUF
#define PARBA_NBUF 2
#endif
// narrow store flush of interior tiles: 256-bit stores of edge pairs (A/B
// knob; measured 2.1% slower at C2 than 128-bit rows, profiles/r02_ab_st256.txt: off)
#ifndef PARBA_ST256
#define PARBA_ST256 0
#endif
constexpr int kStageBufs = PARBA_NBUF;

constexpr int kThreads = kWarps * 32;
// Warps per CTA of the streaming sinks (window, full, targets); with
// PARBA_MINB_STREAM = 2 two such CTAs share an SM (A/B knob).
#ifndef PARBA_WARPS_STREAM
#define PARBA_WARPS_STREAM 32
#endif

// kTargets: the full histogram's first pass — each warp appends the u32
// targets it finishes to its own region of a scratch buffer (order is
// irrelevant to a histogram); parba_hist.cuh partitions and counts them.
// kTargetsK: the same for a window, keeping only targets < klim.
// kStoreT: store mode emitting only the u32 target of each edge, in edge
// order (tgt[i - lo]); the source is a closed form the host fills in
// (parba_host.cu: the end-to-end host-array path moves 4 B per edge over
// PCIe instead of 16).
enum SinkKind { kStore = 0, kWindow = 1, kFull = 2, kTargets = 3, kTargetsK = 4, kStoreT = 5 };
constexpr int kSinkKinds = 6;
__host__ __device__ constexpr bool is_targets(int sink) { return sink == kTargets || sink == kTargetsK; }
__host__ __device__ constexpr bool is_store(int sink) { return sink == kStore || sink == kStoreT; }
__host__ __device__ constexpr int warps_for(int sink) { return is_store(sink) ? kWarps : PARBA_WARPS_STREAM; }
#ifndef PARBA_HIST_BUCKETS
#define PARBA_HIST_BUCKETS 2048
#endif
// buckets one scatter pass handles (parba_hist.cuh); a target domain of up
// to kHistBucketsMax buckets is scattered in several passes
constexpr int kHistBuckets = PARBA_HIST_BUCKETS;
#ifndef PARBA_HIST_BUCKETS_MAX
#define PARBA_HIST_BUCKETS_MAX 8192
#endif
constexpr int kHistBucketsMax = PARBA_HIST_BUCKETS_MAX;  // targets sink: bucket histogram per warp group
constexpr int kBucketBits = 13;        // bucket field of a count work item
#ifndef PARBA_HIST_GROUPS
#define PARBA_HIST_GROUPS 1
#endif
constexpr int kHistGroups = PARBA_HIST_GROUPS;  // warp groups (scatter CTAs) per tile CTA

#ifndef PARBA_WARP_TIMES
#define PARBA_WARP_TIMES 0
#endif
#if PARBA_WARP_TIMES
// diagnostic build: start/end globaltimer of every warp of the last launch
constexpr uint64_t kMaxTimedWarps = 148 * 32;
__device__ unsigned long long g_warp_times[2 * kMaxTimedWarps];
#endif

struct SinkArgs {
    uint64_t *out;                         // store: 2*(hi-lo) u64, 16-byte aligned
    unsigned long long *win;               // window counts (K)
    uint32_t *full;                        // full counts (n)
    uint32_t *t32;                         // targets: capw u32 slots per warp
    uint64_t capw;
    uint32_t *hist;                        // targets: H[b * G * gridDim.x + G * blk + group]
    int shift, nb;                         //   (bucket = target >> shift, G = kHistGroups)
    Magic32 bdiv;                          // targets / store-targets histogram: bucket = target / bucket width
    uint64_t klim;                         // targets: only targets < klim are kept
    int by_pos;                            // targets, degree sequence: emit positions (full counts)
    uint64_t t32_cap;                      // host side: slots of t32
    uint64_t *t32_geom;                    // host side: {slots filled, capw, warps per CTA, CTAs, tile edges}
};

// Shared-memory layout of a tile CTA (dynamic smem, W warps):
//   [pad][queue 0] .. [queue W-1] [CRC tables][crc(0,2j+1)] [stage 0] .. [stage W-1] [slots]
// Each warp's pending queue is a ring of kQueue entries of kEB bytes aligned
// to its own size kQB, so an entry address is qbase | (cursor & (kQB - 1))
// with byte cursors.  Store-mode entries carry the chain value and where its
// terminal value goes (the stage cell):
//   narrow (values < 2^32):  (smem address of the cell << 32) | value
//   kPack  (values < 2^52):  (cell offset in the warp's stage << 52) | value
//   otherwise:               value, offsets in a separate u16 ring (slots).
// The stage holds the terminal values of the two tiles in flight.
template <class Hash, int SINK>
struct TileLayout {
    using R = typename Hash::R;
    static constexpr uint32_t kEB = is_store(SINK) ? 8u : (uint32_t)sizeof(R);
    static constexpr uint32_t kLgEB = kEB == 8 ? 3u : 2u;
    // wide store (64-bit values, packed entries): a 256-entry queue, with
    // phase 1 split in two halves and a drain between them (at most 31 + 128
    // entries are ever queued), so 32 warps fit instead of 23
    // 512-edge tiles: narrow CRC store and store-targets kernels (the stage of
    // a wide one would not fit), optionally the streaming sinks (no stage; the
    // queue stays 512 entries with a drain after 256 edges)
    static constexpr bool kBig =
        Hash::kHasCrc && ((PARBA_TILE512 && SINK == kStore && Hash::kNarrow) ||
                          (PARBA_TILE512_ST && SINK == kStoreT && Hash::kNarrow) ||
                          (PARBA_TILE512_STREAM && !is_store(SINK)));
    static constexpr int kTileE = kBig ? 2 * kTile : kTile;  // edges per warp tile of this kernel
    static constexpr int kEplE = kTileE / 32;                 // edges per lane in phase 1
    static constexpr bool kSplit =
        is_store(SINK) && (kBig || (!Hash::kNarrow && Hash::kPack && PARBA_WIDE_SPLIT) ||
                           (Hash::kNarrow && PARBA_NARROW_SPLIT));
    // edges per lane between two drains: 4 with the 256-entry queue of a split
    // store kernel, else 8 (the whole 256-edge tile, half a 512-edge one)
    static constexpr int kPieceEpl = kSplit ? PARBA_PIECE : 8;
    static constexpr uint32_t kQ = kSplit ? 256u : (uint32_t)kQueue;
    static constexpr uint32_t kQB = kQ * kEB;
    static constexpr uint32_t kTB = kTileE * (uint32_t)sizeof(R);  // one stage buffer
    static constexpr uint32_t kStageB = is_store(SINK) ? kStageBufs * kTB : 0;
    static constexpr bool kSlots = is_store(SINK) && !Hash::kPack;
    static constexpr uint32_t kSlotB = kSlots ? kQueue * 2 : 0;
    static constexpr size_t kTabB = Hash::kHasCrc ? (Hash::kTableWords + kTileE) * 4 : 0;
    static constexpr size_t kHistB = is_targets(SINK)   ? kHistGroups * kHistBucketsMax * 4
                                     : SINK == kStoreT ? kHistBuckets * 4
                                                       : 0;
    static constexpr size_t kWinB = SINK == kWindow ? kWinSmem * 4 : 0;
    static constexpr size_t fixed = kQB /* alignment pad */ + kTabB + kHistB + kWinB;
    static constexpr size_t per_warp = kQB + kStageB + kSlotB;
};
constexpr uint64_t kValueMask52 = (1ull << 52) - 1;
// Byte cursors of one launch stay below 2^31 when a launch covers at most
// kLaunchEdgesPerWarp edges per warp (the host splits larger ranges).
constexpr uint64_t kLaunchEdgesPerWarp = 1ull << 27;

// Window sink, optional shared-memory privatisation (the north star's
// suggestion; A/B knob PARBA_WIN_SMEM, off): the counts of the lowest nodes --
// the hottest part of the window, node v draws ~1/sqrt(v) of the targets --
// live in a per-CTA u32 array in shared memory and are added to the global
// window once at the end of the launch.  Measured at C3: 8K bins -1.8%, 16K
// bins -4.8% (the bins cost resident warps; only ~2% of edges hit the window
// and its 800 KB stay in L2), profiles/r02_ab_window_smem_and_unroll.txt.

__device__ __forceinline__ void win_add(const SinkArgs &a, uint32_t wsm, uint64_t t) {
#if PARBA_WIN_SMEM > 0
    if (t < kWinSmem) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(wsm + 4u * (uint32_t)t) : "memory");
        return;
    }
#endif
    atomicAdd(a.win + t, 1ull);
}

// A chain finished with terminal value r: hand its target to the sink.
template <bool NARROW, bool SEED, int SINK, class R, bool DEG = false>
__device__ __forceinline__ void finish(uint32_t saddr, uint64_t r, const DevParams &p, const SinkArgs &a,
                                       uint32_t wsm = 0) {
    if constexpr (is_store(SINK)) {
        sts_t<R>(saddr, (R)r);  // stage cell; the target is computed at flush
    } else if constexpr (SINK == kWindow) {
        if (SEED && r < p.stop) {
            const uint64_t t = __ldg(p.seed + r);
            if (t < p.K) win_add(a, wsm, t);
        } else if (NARROW ? ((uint32_t)r < p.win_rlim32) : (r < p.win_rlim)) {
            // generated target < K  <=>  r < win_rlim (wide: the FP64 reciprocal
            // instead of a 64-bit division when the host allows it)
            if constexpr (!NARROW && !DEG) {
                if (p.win_fp) {
                    win_add(a, wsm, target_fp<SEED>(r, p));
                    return;
                }
            }
            win_add(a, wsm, source_of<NARROW, SEED, DEG>(r >> 1, p));
        }
    } else {
        atomicAdd(a.full + target_of<NARROW, SEED, false, DEG>(r, p), 1u);
    }
}

template <class Hash, int SINK, bool SEED, bool DEG = false>
__global__ void __launch_bounds__(32 * warps_for(SINK), is_store(SINK) ? PARBA_MINB_STORE : PARBA_MINB_STREAM)
tile_kernel(DevParams p, uint64_t lo, uint64_t hi, uint64_t tile0, uint64_t ntiles,
            SinkArgs a, unsigned long long *probes_out) {
    using R = typename Hash::R;
    constexpr bool NARROW = Hash::kNarrow;
    using L = TileLayout<Hash, SINK>;
    constexpr int kTile = L::kTileE;  // this kernel's tile (shadows the default)
    // one-stage first probes: per hash class, and for every store kernel up to 5 chunks
    constexpr bool kRy1 = Hash::kHasRy1 || (is_store(SINK) && Hash::kHasRy1Store);
    constexpr int kEpl = L::kEplE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;  // warps per CTA (<= kWarps; fewer when smem is tight)
    // queues first, each aligned to its size (the launch reserves kQB of padding)
    const uint32_t raw_s = smem_addr(smem_raw);
    const uint32_t pad = (L::kQB - (raw_s & (L::kQB - 1))) & (L::kQB - 1);
    unsigned char *tab_raw = smem_raw + pad + (size_t)wpc * L::kQB;
    uint32_t *tabs_p = reinterpret_cast<uint32_t *>(tab_raw);
    uint32_t *clow_s = tabs_p + Hash::kTableWords;  // crc(0, 2j+1), j < kTile (2j+1 < 512)
    const uint32_t tabs = opaque(smem_addr(tabs_p));
    if constexpr (Hash::kHasCrc) {
        // the 64 single-bit CRCs in queue 0's space (unused until phase 1);
        // every table entry and crc(0, 2j+1) is an XOR of them
        uint32_t *bits = reinterpret_cast<uint32_t *>(smem_raw + pad);
        Hash::build_linear(tabs_p, bits, p.k0);
        for (int j = threadIdx.x; j < kTile; j += blockDim.x) {
            uint32_t x = 2u * (uint32_t)j + 1u, v = 0u;
            while (x) {
                v ^= bits[__ffs(x) - 1];
                x &= x - 1;
            }
            clow_s[j] = v;
        }
    }
    // targets sink: the CTA's bucket histograms follow the stage and slot
    // areas, i.e. the last kHistB bytes of the layout
    [[maybe_unused]] uint32_t *hist_s = reinterpret_cast<uint32_t *>(
        smem_raw + pad + (size_t)wpc * (L::kQB + L::kStageB + L::kSlotB) + L::kTabB);
    if constexpr (is_targets(SINK))
        for (int b = threadIdx.x; b < kHistGroups * a.nb; b += blockDim.x) hist_s[b] = 0;
    if constexpr (SINK == kStoreT)
        if (a.hist)
            for (int b = threadIdx.x; b < a.nb; b += blockDim.x) hist_s[b] = 0;
    // window sink: privatised bins after the stage/slot areas (kWinB bytes)
    [[maybe_unused]] uint32_t *win_s = reinterpret_cast<uint32_t *>(
        smem_raw + pad + (size_t)wpc * (L::kQB + L::kStageB + L::kSlotB) + L::kTabB);
    [[maybe_unused]] uint32_t wsm = 0;
#if PARBA_WIN_SMEM > 0
    if constexpr (SINK == kWindow) {
        for (uint32_t b = threadIdx.x; b < kWinSmem; b += blockDim.x) win_s[b] = 0;
        wsm = opaque(smem_addr(win_s));
    }
#endif
    __syncthreads();

    // shared-window addresses of this warp's queue, stage and slot ring
    const uint32_t qbase = opaque(raw_s + pad + (uint32_t)wib * L::kQB);
    const uint32_t st_all = raw_s + pad + (uint32_t)wpc * L::kQB + (uint32_t)L::kTabB;
    [[maybe_unused]] const uint32_t stage_s = opaque(st_all + (uint32_t)wib * L::kStageB);
    [[maybe_unused]] const uint32_t qs_s =
        opaque(st_all + (uint32_t)wpc * L::kStageB + (uint32_t)wib * L::kSlotB);
    const unsigned ltmask = lanemask_lt();
#if PARBA_WARP_TIMES
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    const uint64_t gw = (uint64_t)blockIdx.x * wpc + wib;
    const uint64_t nw = (uint64_t)gridDim.x * wpc;

    // NS chains per lane in phase 2 (independent probes for the scheduler)
    constexpr int NS = is_store(SINK) ? PARBA_ILP_STORE : is_targets(SINK) ? PARBA_ILP_TARGETS : PARBA_ILP_STREAM;
    uint32_t act[NS];               // 1: slot holds a running chain
    R r[NS];
    uint32_t saddr[NS];             // store: smem address of the chain's stage cell
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        act[q] = 0;
        r[q] = 0;
        saddr[q] = 0;
    }
    uint32_t headb = 0, tailb = 0;  // queue byte cursors (warp-uniform)
    uint32_t tile_q0 = 0;           // tail cursor at the start of the current tile
    uint32_t probes = 0;            // per lane (< 2^32 per launch and lane)
    uint64_t prev_base = 0;         // base of the tile the next flush writes
    bool have_prev = false;
    uint32_t buf = 0;               // stage buffer of the current tile
    [[maybe_unused]] uint64_t mid_base = 0;  // 3 buffers: base of tile t-1
    [[maybe_unused]] uint32_t q0_prev = 0;   // 3 buffers: queue cursor at the start of tile t-1
    [[maybe_unused]] uint32_t n_inflight = 0;

    auto qaddr = [&](uint32_t cur) -> uint32_t { return qbase | (cur & (L::kQB - 1)); };

    auto is_done = [&](R v) -> bool {
        if constexpr (SEED) return ((uint32_t)v & 1u) == 0 || (uint64_t)v < p.stop;
        else return ((uint32_t)v & 1u) == 0;
    };

    // Write a finished tile out of buffer b (store mode): (source, target)
    // pairs from the staged terminal values, 16-byte streaming stores.
    // Interior tiles (all but the range ends) skip the per-edge bounds test.
    auto flush_t = [&](auto full_c, uint32_t b, uint64_t base) {
        [[maybe_unused]] constexpr bool FULL = decltype(full_c)::value;
        if constexpr (SINK == kStoreT) {
            // targets only (n < 2^32): 4 B per edge, 128 B per warp store.
            // Histogram mode (a.hist, the full-histogram count): slot i -
            // tile0*kTile (tile order, grid-stride tiles as always, so every
            // CTA sees a representative mix of the batch), empty slots for
            // positions outside [lo, hi), and bucket = target >> shift
            // counted in the CTA's histogram; the scatter reads a CTA's tiles
            // as every nw-th run of wpc tiles.
            // wide launches: targets by the FP64 reciprocal when allowed
            auto tgt_at = [&](auto fp_c, uint32_t j) -> uint32_t {
                const uint64_t r = (uint64_t)lds_t<R>(stage_s + (b * kTile + j) * (uint32_t)sizeof(R));
                if constexpr (!NARROW && decltype(fp_c)::value) return (uint32_t)target_fp<SEED>(r, p);
                else return (uint32_t)target_of<NARROW, SEED, Hash::kR31, false>(r, p);
            };
            auto rows = [&](auto fp_c) {
                if (a.hist) {
                    uint32_t *o = a.t32 + (int64_t)(base - tile0 * kTile);
#pragma unroll
                    for (int k = 0; k < kEpl; ++k) {
                        const uint32_t j = lane + 32u * k;
                        const uint64_t i = base + j;
                        uint32_t tg = 0xffffffffu;
                        if (FULL || (i >= lo && i < hi)) {
                            tg = tgt_at(fp_c, j);
                            atomicAdd(hist_s + (uint32_t)(((uint64_t)tg * a.bdiv.mul) >> a.bdiv.shift), 1u);
                        }
                        __stcs(o + j, tg);
                    }
                    return;
                }
                uint32_t *o = a.t32 + (int64_t)(base - lo);
#pragma unroll
                for (int k = 0; k < kEpl; ++k) {
                    const uint32_t j = lane + 32u * k;
                    const uint64_t i = base + j;
                    if (FULL || (i >= lo && i < hi)) __stcs(o + j, tgt_at(fp_c, j));
                }
            };
            if (!NARROW && p.tgt_fp) rows(std::true_type{});
            else rows(std::false_type{});
        } else if constexpr (SINK == kStore) {
            ulonglong2 *o = reinterpret_cast<ulonglong2 *>(a.out) + (int64_t)(base - lo);
            if constexpr (FULL && !NARROW && !DEG) {
                // 64-bit positions: one 64-bit division per lane and tile, then
                // the lane's 8 sources from the remainder by the 32-bit magic
                // (remainder + 32k < d + 224 < 2^31)
                if (p.d < (1ull << 30)) {
                    const uint64_t i0 = base + lane - (SEED ? p.m0 : 0);
                    const uint64_t q0 = magic_div(i0, p.div64) + (SEED ? p.n0 : 0);
                    const uint32_t r0 = (uint32_t)(i0 - (q0 - (SEED ? p.n0 : 0)) * p.d);
                    // targets: FP64 reciprocal (target_fp: one DFMA instead of
                    // a 64-bit multiply-high division) when the host allows it
                    auto rows = [&](auto fp_c) {
#pragma unroll
                        for (int k = 0; k < kEpl; ++k) {
                            const uint32_t j = lane + 32u * k;
                            const uint64_t r = (uint64_t)lds_t<R>(stage_s + (b * kTile + j) * (uint32_t)sizeof(R));
                            uint64_t tgt;
                            if constexpr (decltype(fp_c)::value) tgt = target_fp<SEED>(r, p);
                            else tgt = target_of<NARROW, SEED, false, false>(r, p);
                            __stcs(o + j, make_ulonglong2(q0 + magic_div32(r0 + 32u * k, p.div32), tgt));
                        }
                    };
                    if (p.tgt_fp) rows(std::true_type{});
                    else rows(std::false_type{});
                    return;
                }
            }
#if PARBA_ST256
            if constexpr (FULL && NARROW && !DEG) {
                // interior tile, 32-byte aligned rows: each lane writes pairs of
                // consecutive edges (2*lane + 64k, +1) with one 256-bit store,
                // their two staged values read by one 8-byte load
                if ((reinterpret_cast<uintptr_t>(o) & 31u) == 0) {
#pragma unroll
                    for (int k = 0; k < kEpl / 2; ++k) {
                        const uint32_t j = 2u * lane + 64u * k;
                        const uint64_t i = base + j;
                        const uint64_t rr = lds_u64(stage_s + (b * kTile + j) * 4u);
                        const uint64_t t0 = target_of<NARROW, SEED, Hash::kR31, false>((uint64_t)(uint32_t)rr, p);
                        const uint64_t t1 = target_of<NARROW, SEED, Hash::kR31, false>(rr >> 32, p);
                        stcs_256(o + j, source_of<NARROW, SEED, false>(i, p), t0,
                                 source_of<NARROW, SEED, false>(i + 1, p), t1);
                    }
                    return;
                }
            }
#endif
#pragma unroll
            for (int k = 0; k < kEpl; ++k) {
                const uint32_t j = lane + 32u * k;
                const uint64_t i = base + j;
                if (FULL || (i >= lo && i < hi)) {
                    const uint64_t tgt = target_of<NARROW, SEED, Hash::kR31 && !DEG, DEG>(
                        (uint64_t)lds_t<R>(stage_s + (b * kTile + j) * (uint32_t)sizeof(R)), p);
                    __stcs(o + j, make_ulonglong2(source_of<NARROW, SEED, DEG>(i, p), tgt));
                }
            }
        }
    };
    auto flush = [&](uint32_t b, uint64_t base) {
        if constexpr (is_store(SINK)) {
            __syncwarp();
            if (base >= lo && base + kTile <= hi) flush_t(std::true_type{}, b, base);
            else flush_t(std::false_type{}, b, base);
            __syncwarp();
        }
    };

    // targets sink: the warp's finished targets go to consecutive slots of its
    // region (one ballot per step, so a warp's stores are contiguous)
    [[maybe_unused]] uint32_t *wout = nullptr;
    [[maybe_unused]] uint32_t wcur = 0;
    [[maybe_unused]] uint32_t *hist_w = hist_s;  // this warp's group
    if constexpr (is_targets(SINK)) {
        wout = a.t32 + gw * a.capw;
        hist_w = hist_s + (uint32_t)(wib * kHistGroups / wpc) * a.nb;
    }
    // targets >= klim (full: n; window: the K lowest nodes) are dropped
    auto emit = [&](bool f, uint64_t rv) {
        if constexpr (is_targets(SINK)) {
            if constexpr (SINK == kTargets && DEG) {
                if (a.by_pos) {
                    // degree sequence, full histogram by position: the terminal
                    // position r >> 1 (owner resolved in order by the count
                    // kernel) instead of a random owner lookup here; seed-graph
                    // targets (rare) are counted directly
                    const bool seedt = f && rv < p.stop;
                    if (seedt) atomicAdd(a.full + __ldg(p.seed + rv), 1u);
                    const bool keep = f && !seedt;
                    const unsigned m = ballot_all(keep);
                    if (keep) {
                        const uint32_t e = (uint32_t)(rv >> 1);
                        wout[wcur + __popc(m & ltmask)] = e;
                        atomicAdd(hist_w + (e >> a.shift), 1u);
                    }
                    wcur += __popc(m);
                    return;
                }
            }
            if constexpr (SINK == kTargets) {  // full histogram: every target is kept
                const unsigned m = ballot_all(f);
                if (f) {
                    const uint32_t tg = (uint32_t)target_of<NARROW, SEED, false, DEG>(rv, p);
                    wout[wcur + __popc(m & ltmask)] = tg;
                    atomicAdd(hist_w + (uint32_t)(((uint64_t)tg * a.bdiv.mul) >> a.bdiv.shift), 1u);
                }
                wcur += __popc(m);
            } else {
                uint64_t tg = 0;
                if (f) tg = target_of<NARROW, SEED, false, DEG>(rv, p);
                const bool keep = f && tg < a.klim;
                const unsigned m = ballot_all(keep);
                if (keep) {
                    wout[wcur + __popc(m & ltmask)] = (uint32_t)tg;
                    atomicAdd(hist_w + (uint32_t)(((uint64_t)(uint32_t)tg * a.bdiv.mul) >> a.bdiv.shift), 1u);
                }
                wcur += __popc(m);
            }
        }
    };

    // One probe on every lane (idle lanes hash a harmless stale value and
    // discard it: no divergent branch around the probe); finished chains go
    // to the sink.
    auto step = [&]() {
        R nr[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) nr[q] = Hash::probe(tabs, r[q], p);
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            probes += act[q];
            uint32_t cont = (uint32_t)nr[q] & 1u;  // odd: the chain continues
            if constexpr (SEED) cont &= (uint64_t)nr[q] >= p.stop ? 1u : 0u;
            const uint32_t fin = act[q] & (cont ^ 1u);
            act[q] &= cont;
            r[q] = nr[q];
            if constexpr (is_targets(SINK)) {
                emit(fin != 0, (uint64_t)nr[q]);
            } else if (fin) {
                if constexpr (is_store(SINK)) PARBA_CHECK(saddr[q] - stage_s < L::kStageB);
                finish<NARROW, SEED, SINK, R, DEG>(saddr[q], (uint64_t)nr[q], p, a, wsm);
            }
        }
    };

    // Pop queued chains into idle lanes of slot Q.  FULLQ: at least 32
    // entries queued, so every idle lane takes one (no availability test).
    auto refill1 = [&](auto fullq_c, auto slot_c) {
        constexpr bool FULLQ = decltype(fullq_c)::value;
        constexpr int Q = decltype(slot_c)::value;
        const unsigned idle = ballot_all(!act[Q]);
        const uint32_t rank = __popc(idle & ltmask);
        const uint32_t availb = tailb - headb;
        if (!act[Q] && (FULLQ || (rank << L::kLgEB) < availb)) {
            const uint32_t cur = headb + (rank << L::kLgEB);
            if constexpr (is_store(SINK)) {
                const uint64_t e = lds_u64(qaddr(cur));
                if constexpr (NARROW) {
                    r[Q] = (R)(uint32_t)e;
                    saddr[Q] = (uint32_t)(e >> 32);
                } else if constexpr (Hash::kPack) {
                    r[Q] = (R)(e & kValueMask52);
                    saddr[Q] = stage_s + (uint32_t)(e >> 52) * (uint32_t)sizeof(R);
                } else {
                    r[Q] = (R)e;
                    saddr[Q] = stage_s + lds_u16(qs_s + ((cur & (L::kQB - 1)) >> 2));
                }
            } else {
                r[Q] = lds_t<R>(qaddr(cur));
            }
            act[Q] = 1;
        }
        if constexpr (FULLQ) headb += (uint32_t)__popc(idle) << L::kLgEB;
        else headb += min((uint32_t)__popc(idle) << L::kLgEB, availb);
    };
    auto refill = [&](auto fullq_c) {
        refill1(fullq_c, std::integral_constant<int, 0>{});
        if constexpr (NS > 1) refill1(fullq_c, std::integral_constant<int, 1>{});
    };
    auto any_act = [&]() -> bool {
        uint32_t x = 0;
#pragma unroll
        for (int q = 0; q < NS; ++q) x |= act[q];
        return __any_sync(0xffffffffu, x);
    };

    // RY = 1: large tile (2*base >= kRyMin): the lane's 8 start values differ by
    // multiples of 64, so 1/r0 comes from one reciprocal per lane and tile,
    // c = 1/rc at the centre rc, and the first-order series
    // 1/(rc + e) ~ c - e*c^2 (relative error (e/rc)^2 < 2^-38 for |e| <= 224).
    // RY = 2: 2-chunk tiles with 2*base >= kOneStageMin take the same series
    // into the one-stage remainder (mod_fp31_y1: no rd, 4 FP64 instructions
    // instead of 7 per first probe).
    [[maybe_unused]] double rc = 0.0, c = 0.0, s64 = 0.0;  // RY: this lane's series of the current tile
    auto ry_setup = [&](uint64_t base, int half) {  // half: the lane's edges 8*half .. 8*half + 7
        rc = u52_to_f64(2 * base + 2 * lane + 1 + 224 + 512 * half);
        c = recip_approx(rc);
        s64 = 64.0 * c * c;
    };
    // first probes of the lane's edges k in [KB, KE) of the tile
    auto phase1 = [&](auto full_c, auto ry_c, uint64_t base, uint32_t cb, auto kb_c, auto ke_c) {
        constexpr bool FULL = decltype(full_c)::value;
        constexpr int RY = decltype(ry_c)::value;  // 0: none, 1: series, 2: series + one-stage remainder
        constexpr int KB = decltype(kb_c)::value, KE = decltype(ke_c)::value;
#pragma unroll
        for (int k = KB; k < KE; ++k) {
            const uint32_t j = lane + 32u * k;
            const uint64_t i = base + j;
            const bool valid = FULL || ((i >= lo) && (i < hi));
            const R r0 = (R)(2 * base) + (R)(2 * j + 1);
            R r1;
            if constexpr (RY == 2) {
                if constexpr (kRy1)
                    r1 = Hash::from_crc_ry1(cb ^ clow_s[j], r0, fma(-((k & 7) - 3.5), s64, c), p);
            } else if constexpr (RY == 1) {
                static_assert(kEpl % 8 == 0, "one series centre per 8 edges of a lane");
                const double e = 64.0 * (k & 7) - 224.0;
                r1 = Hash::from_crc_ry(cb ^ clow_s[j], r0, rc + e, fma(-((k & 7) - 3.5), s64, c), p);
            } else if constexpr (Hash::kHasCrc) {
                r1 = Hash::from_crc(cb ^ clow_s[j], r0, p);
            } else {
                r1 = Hash::probe(tabs, r0, p);
            }
            const bool done = is_done(r1);
            [[maybe_unused]] const uint32_t cell = stage_s + (buf * kTile + j) * (uint32_t)sizeof(R);
            if constexpr (is_store(SINK))  // final unless pending
                sts_t<R>(cell, r1);
            if constexpr (is_targets(SINK)) emit(valid && done, (uint64_t)r1);
            else if constexpr (!is_store(SINK)) if (valid && done) finish<NARROW, SEED, SINK, R, DEG>(0u, (uint64_t)r1, p, a, wsm);
            const bool pend = valid && !done;
            const unsigned m = ballot_all(pend);
            const uint32_t cur = tailb + (__popc(m & ltmask) << L::kLgEB);
            if constexpr (is_store(SINK)) {
                if constexpr (NARROW) {
                    sts_u64_if(pend, qaddr(cur), ((uint64_t)cell << 32) | (uint64_t)r1);
                } else if constexpr (Hash::kPack) {
                    sts_u64_if(pend, qaddr(cur), ((uint64_t)(buf * kTile + j) << 52) | (uint64_t)r1);
                } else if (pend) {
                    sts_u64(qaddr(cur), (uint64_t)r1);
                    sts_u16(qs_s + ((cur & (L::kQB - 1)) >> 2), (uint16_t)(cell - stage_s));
                }
            } else {
                sts_t_if<R>(pend, qaddr(cur), r1);
            }
            tailb += __popc(m) << L::kLgEB;
            PARBA_CHECK(tailb - headb <= L::kQB);  // the ring never overflows
            probes += valid ? 1u : 0u;
        }
    };

    for (uint64_t t = gw; t < ntiles; t += nw) {
        const uint64_t base = (tile0 + t) * kTile;
        // ---- phase 1: first probe of all edges of the tile
        tile_q0 = tailb;  // queue position where this tile's entries start
        uint32_t cb = 0;
        if constexpr (Hash::kHasCrc) cb = Hash::crc(tabs, 2 * base, p);
        // ---- phase 2 body: pop queued chains into idle lanes and probe while
        // at least a full warp of entries is queued (the < 32 newest entries
        // carry over, so every refill can fill every idle lane)
        auto drain = [&]() {
#if PARBA_P2_UNROLL >= 2
            // two refill+probe steps per loop test while >= 2 warps of entries wait
            if ((is_store(SINK) || PARBA_P2_UNROLL_STREAM) && tailb - headb >= ((64u * NS) << L::kLgEB)) {
                const uint32_t lim2 = tailb - ((64u * NS) << L::kLgEB);
                do {
                    refill(std::true_type{});
                    step();
                    refill(std::true_type{});
                    step();
                } while (headb <= lim2);
            }
#endif
            if (tailb - headb >= ((32u * NS) << L::kLgEB)) {
                const uint32_t lim = tailb - ((32u * NS) << L::kLgEB);
                do {
                    refill(std::true_type{});
                    step();
                } while (headb <= lim);
            }
        };
        // phase 1 over all 8 edges per lane, or in two halves with a drain
        // between them (the 256-entry queue of the wide store)
        auto run_phase1 = [&](auto full_c, auto ry_c) {
            constexpr int PE = L::kPieceEpl, NP = kEpl / PE;
            static_assert(NP * PE == kEpl && NP <= 8 && (8 % PE == 0 || PE % 8 == 0), "phase-1 pieces");
            // piece P: the lane's edges [P*PE, (P+1)*PE); a new reciprocal
            // series at every 8th edge; a drain between pieces
            auto piece = [&](auto p_c) {
                constexpr int P = decltype(p_c)::value;
                if constexpr (P < NP) {
                    if constexpr (decltype(ry_c)::value != 0 && (P * PE) % 8 == 0) ry_setup(base, (P * PE) / 8);
                    if constexpr (P > 0) {
                        // the next piece pushes at most 32 * PE entries: drain only
                        // when the ring could not take them (larger drains run more
                        // of their steps in the unrolled loop)
                        __syncwarp();
#if PARBA_LAZY_DRAIN
                        if (tailb - headb > ((L::kQ - 32u * PE) << L::kLgEB)) drain();
#else
                        drain();
#endif
                    }
                    phase1(full_c, ry_c, base, cb, std::integral_constant<int, P * PE>{},
                           std::integral_constant<int, (P + 1) * PE>{});
                }
            };
            piece(std::integral_constant<int, 0>{});
            piece(std::integral_constant<int, 1>{});
            piece(std::integral_constant<int, 2>{});
            piece(std::integral_constant<int, 3>{});
            piece(std::integral_constant<int, 4>{});
            piece(std::integral_constant<int, 5>{});
            piece(std::integral_constant<int, 6>{});
            piece(std::integral_constant<int, 7>{});
        };
        if (base >= lo && base + kTile <= hi) {
            using I0 = std::integral_constant<int, 0>;
            using I1 = std::integral_constant<int, 1>;
            using I2 = std::integral_constant<int, 2>;
            if constexpr (kRy1) {
                if (2 * base >= kOneStageMin) run_phase1(std::true_type{}, I2{});
                else if (2 * base >= kRyMin) run_phase1(std::true_type{}, I1{});
                else run_phase1(std::true_type{}, I0{});
            } else if constexpr (Hash::kHasRy) {
                if (2 * base >= kRyMin) run_phase1(std::true_type{}, I1{});
                else run_phase1(std::true_type{}, I0{});
            } else {
                run_phase1(std::true_type{}, I0{});
            }
        } else {
            run_phase1(std::false_type{}, std::integral_constant<int, 0>{});
        }
        __syncwarp();
        // the end-of-tile drain is lazy too (PARBA_LAZY_END; bit 0: store
        // sinks, bit 1: streaming sinks): entries stay queued while the ring
        // can still take the next tile's first piece
        if constexpr (((PARBA_LAZY_END & 1) && is_store(SINK) && L::kSplit) || ((PARBA_LAZY_END & 2) && !is_store(SINK))) {
            if (tailb - headb > ((L::kQ - 32u * L::kPieceEpl) << L::kLgEB)) drain();
        } else {
            drain();
        }
        // ---- store: flush the oldest tile in flight once none of its chains runs
        if constexpr (is_store(SINK)) {
            if (have_prev) {
                // oldest tile: t-1 (2 buffers) or t-2 (3 buffers)
                const uint32_t pb = kStageBufs == 2 ? (buf ^ 1u) : (buf == 2 ? 0u : buf + 1);
                const uint32_t q_end = kStageBufs == 2 ? tile_q0 : q0_prev;  // its entries end here
                // entries of that tile still queued: pop them first
                while ((int32_t)(q_end - headb) > 0) {
                    refill(std::false_type{});
                    step();
                }
                for (;;) {
                    uint32_t x = 0;
#pragma unroll
                    for (int q = 0; q < NS; ++q) x |= act[q] & ((saddr[q] - stage_s) / L::kTB == pb ? 1u : 0u);
                    if (!__any_sync(0xffffffffu, x)) break;
                    // keep the lanes that are free busy with this tile's chains
                    if (tailb != headb) refill(std::false_type{});
                    step();
                }
                flush(pb, prev_base);
            }
            if constexpr (kStageBufs == 2) {
                prev_base = base;
                have_prev = true;
                buf ^= 1u;
            } else {
                have_prev = n_inflight >= 1;  // tile t-1 will be the next tile's t-2
                if (n_inflight < 2) ++n_inflight;
                prev_base = mid_base;         // t-1 becomes the oldest
                mid_base = base;
                q0_prev = tile_q0;
                buf = buf == 2 ? 0u : buf + 1;
            }
        }
    }
    // ---- drain the queue and the chains still running, then flush the last tile
    while (tailb != headb) {
        refill(std::false_type{});
        step();
    }
    while (any_act()) step();
    if constexpr (is_targets(SINK)) {  // unused slots of the region: empty
        PARBA_CHECK(wcur <= a.capw);
        for (uint64_t j = wcur + lane; j < a.capw; j += 32) wout[j] = 0xffffffffu;
        __syncthreads();
        for (int i = threadIdx.x; i < kHistGroups * a.nb; i += blockDim.x) {
            const int g = i / a.nb, b = i - g * a.nb;
            a.hist[(uint64_t)b * kHistGroups * gridDim.x + (uint64_t)kHistGroups * blockIdx.x + g] = hist_s[i];
        }
    }
#if PARBA_WIN_SMEM > 0
    if constexpr (SINK == kWindow) {  // privatised bins -> the global window
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < kWinSmem && b < p.K; b += blockDim.x)
            if (win_s[b]) atomicAdd(a.win + b, (unsigned long long)win_s[b]);
    }
#endif
    if constexpr (is_store(SINK)) {
        if constexpr (kStageBufs == 2) {
            if (have_prev) flush(buf ^ 1u, prev_base);
        } else {
            // the last two tiles: buffers buf-2 (older) and buf-1 (newer)
            const uint32_t b1 = buf == 0 ? 2u : buf - 1;
            const uint32_t b2 = b1 == 0 ? 2u : b1 - 1;
            if (n_inflight == 2) flush(b2, prev_base);
            if (n_inflight >= 1) flush(b1, mid_base);
        }
    }
    if constexpr (SINK == kStoreT) {
        if (a.hist) {  // the CTA's bucket histogram (its tiles: every nw-th run of wpc tiles)
            __syncthreads();
            for (int b = threadIdx.x; b < a.nb; b += blockDim.x)
                a.hist[(uint64_t)b * gridDim.x + blockIdx.x] = hist_s[b];
        }
    }
#if PARBA_WARP_TIMES
    {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        const uint64_t wid = (uint64_t)blockIdx.x * wpc + wib;
        if (lane == 0 && wid < kMaxTimedWarps) {
            g_warp_times[2 * wid] = t_start;
            g_warp_times[2 * wid + 1] = t_end;
        }
    }
#endif
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

template <class Hash, bool DEG = false>
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
                make_ulonglong2(source_of<false, true, DEG>(ids[k], p), target_of<false, true, false, DEG>(r, p));
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

// crc32c_u64_many (hashing.py:158-165): out[k] = crc(seed, words[k]) via
// CRC linearity -- byte tables of crc(0, .) with crc(seed, 0) folded in.
__global__ void __launch_bounds__(256)
crc_kernel(uint32_t k0, const uint64_t *__restrict__ w, uint64_t count, uint64_t *__restrict__ out) {
    __shared__ uint32_t tabs_p[8 * 256];
    build_byte_tables(tabs_p, 8, k0);
    __syncthreads();
    const uint32_t tabs = opaque(smem_addr(tabs_p));
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = crc_bytes<8>(tabs, w[k]);
}

// mulhi_u64 (hashing.py:168-176): high 64 bits of a[k] * b[k].
__global__ void mulhi_kernel(const uint64_t *__restrict__ a, const uint64_t *__restrict__ b, uint64_t count,
                             uint64_t *__restrict__ out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = __umul64hi(a[k], b[k]);
}

// Source endpoints of a window/full count in closed form: node v owns edges
// [m0+(v-n0)d, m0+(v-n0+1)d) (degree sequence: [W[v-n0], W[v-n0+1])); its
// count grows by the overlap with [lo,hi).
template <typename CountT, bool DEG = false>
__global__ void source_counts_kernel(DevParams p, uint64_t lo, uint64_t hi, uint64_t vlo,
                                     uint64_t vhi, CountT *counts) {
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a, b;
        if constexpr (DEG) {
            a = __ldg(p.W + (v - p.n0));
            b = __ldg(p.W + (v - p.n0) + 1);
        } else {
            a = p.m0 + (v - p.n0) * p.d;
            b = a + p.d;
        }
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
