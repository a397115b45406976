// parba_api.cu -- the C ABI core (include/parba_b200.h): validation,
// template dispatch (hash family x CRC width x sink), persistent-grid sizing
// and the device entry points of the plain path.  The node-granular entry
// points live in parba_nodes_api.cu, the host-buffer ones in parba_host.cu.
// No torch types cross this boundary.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/parba_b200.h"
#include "parba_common.h"
#include "parba_kernels.cuh"
#include "parba_hist.cuh"

#include <cub/device/device_scan.cuh>

using namespace parba;
using namespace parba::host;

namespace parba {
namespace host {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int validate(const parba_params_t *p) {
    if (!p) return fail(PARBA_EINVAL, "params is NULL");
    if (p->flags & ~(PARBA_FLAG_NO_SELF_LOOPS | PARBA_FLAG_NO_PARALLEL_EDGES))
        return fail(PARBA_EINVAL, "unknown option flags 0x%x", p->flags);
    if (p->reserved2 != 0) return fail(PARBA_EINVAL, "reserved2 field must be 0");
    if (p->flags && p->m0 < 1)
        return fail(PARBA_EINVAL, "no_self_loops / no_parallel_edges require a seed graph (m0 >= 1): "
                                  "with an empty seed the first edge is the forced self-loop (0, 0)");
    if (is_deg(p)) {
        if (p->d != 0) return fail(PARBA_EINVAL, "exactly one of d and degrees must be given");
        // (a sequence of zero degrees generates nothing and has no directory)
        if (!p->rank && p->m > p->m0) return fail(PARBA_EINVAL, "degree sequence without its rank directory");
        if (p->n < p->n0) return fail(PARBA_EINVAL, "need 0 <= n0 <= n, got n0=%llu, n=%llu",
                                      (unsigned long long)p->n0, (unsigned long long)p->n);
        if (p->hash_kind > PARBA_HASH_SIMPLE) return fail(PARBA_EINVAL, "unknown hash kind %u", p->hash_kind);
        if (p->reserved != 0) return fail(PARBA_EINVAL, "reserved field must be 0");
        if (p->m0 > 0 && !p->seed_edges) return fail(PARBA_EINVAL, "m0 > 0 but seed_edges is NULL");
        if (p->m < p->m0 || p->m >= kMaxEdges)
            return fail(PARBA_EINVAL, "total edge count %llu out of range", (unsigned long long)p->m);
        return PARBA_OK;
    }
    if (p->rank || p->owners) return fail(PARBA_EINVAL, "rank/owners given without a degree sequence");
    if (p->d < 1) return fail(PARBA_EINVAL, "uniform degree must be >= 1, got %llu", (unsigned long long)p->d);
    if (p->n < p->n0) return fail(PARBA_EINVAL, "need 0 <= n0 <= n, got n0=%llu, n=%llu",
                                  (unsigned long long)p->n0, (unsigned long long)p->n);
    if (p->hash_kind > PARBA_HASH_SIMPLE) return fail(PARBA_EINVAL, "unknown hash kind %u", p->hash_kind);
    if (p->reserved != 0) return fail(PARBA_EINVAL, "reserved field must be 0");
    if (p->m0 > 0 && !p->seed_edges) return fail(PARBA_EINVAL, "m0 > 0 but seed_edges is NULL");
    // m = m0 + (n - n0) * d, checked without overflow
    const unsigned __int128 m = (unsigned __int128)p->m0 + (unsigned __int128)(p->n - p->n0) * p->d;
    if (m != p->m) return fail(PARBA_EINVAL, "m=%llu inconsistent with m0 + (n-n0)*d", (unsigned long long)p->m);
    if (p->m >= kMaxEdges) return fail(PARBA_EINVAL, "total edge count %llu exceeds the supported maximum",
                                       (unsigned long long)p->m);
    return PARBA_OK;
}

int check_range(const parba_params_t *p, uint64_t lo, uint64_t hi) {
    if (!(p->m0 <= lo && lo <= hi && hi <= p->m))
        return fail(PARBA_EINVAL, "block [%llu, %llu) out of range [%llu, %llu]", (unsigned long long)lo,
                    (unsigned long long)hi, (unsigned long long)p->m0, (unsigned long long)p->m);
    return PARBA_OK;
}

DevParams make_dev(const parba_params_t *p, uint64_t K) {
    DevParams d{};
    d.n = p->n;
    d.d = p->d;
    d.n0 = p->n0;
    d.m0 = p->m0;
    d.m = p->m;
    d.stop = 2 * p->m0;
    d.mult = p->simple_mult;
    // CRC linearity: crc(s, w) = crc(s, 0) ^ crc(0, w)
    d.k0 = crc32c_u64_bitwise(p->crc_seed0, 0);
    d.k01 = d.k0 ^ crc32c_u64_bitwise(p->crc_seed1, 0);
    d.seed = p->seed_edges;
    const uint64_t dd = p->d ? p->d : 1;  // degree sequences: closed forms unused
    d.div64 = make_magic64(dd);
    d.div32 = make_magic32(dd);
    d.div32_2d = make_magic32(2 * dd);
    d.K = K;
    d.W = p->degree_prefix;
    d.rank = (const ulonglong2 *)p->rank;
    d.owners = p->owners;
    d.dense = p->dense_owner;
    // generated target ((r>>1) - m0)/d + n0 < K  <=>  r < 2*(m0 + (K - n0)*d)
    if (K <= p->n0) {
        d.win_rlim = 0;
    } else {
        const unsigned __int128 lim = 2 * ((unsigned __int128)p->m0 + (unsigned __int128)(K - p->n0) * p->d);
        d.win_rlim = lim > (unsigned __int128)UINT64_MAX ? UINT64_MAX : (uint64_t)lim;
    }
    // narrow launches hold r < 2^32; 2^32-1 is odd, so never a terminal value
    d.win_rlim32 = d.win_rlim > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)d.win_rlim;
    // wide launches: targets by the FP64 reciprocal (target_fp's bounds);
    // PARBA_TGT_FP=0 keeps the 64-bit integer division (A/B)
    const char *tf = getenv("PARBA_TGT_FP");
    d.tgt_fp = (!is_deg(p) && p->d >= 1 && p->d < 174762 && p->n <= (1ull << 32) && !(tf && tf[0] == '0')) ? 1u : 0u;
    d.inv2d = 1.0 / (2.0 * (double)dd);
    // the window sink only resolves targets < K: the same bound holds for any n
    d.win_fp = (!is_deg(p) && p->d >= 1 && p->d < 174762 && K <= (1ull << 32) && !(tf && tf[0] == '0')) ? 1u : 0u;
    return d;
}

}  // namespace host
}  // namespace parba

namespace {

int bits_of(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

// CRC chunk tables needed to cover every chain value of a launch (r <= 2*hi-1,
// the largest first value): 2 -> r < 2^31 (narrow, 32-bit remainder),
// 3 -> r <= kR32Max (0.9375 * 2^32), 4 -> < 2^43, 5 -> < 2^52, 6 -> any.  (Classing by 2*hi
// itself put a range ending at exactly 2^30 edges -- C4's second batch --
// on the slower 3-chunk kernel.)
int nc_for(uint64_t max_r) {
    const int b = bits_of(max_r);
    if (b <= 31) return 2;
    if (PARBA_R32 ? max_r <= kR32Max : b <= 32) return 3;  // the 32-bit tail of mod_fp32_y
    if (b <= 43) return 4;
    if (b <= 52) return 5;
    return 6;
}

struct DevInfo {
    int sms = 0;
    int smem_optin = 0;  // max dynamic shared memory per block
    bool attr_done[12][kSinkKinds][2] = {};  // [hash variant][sink][seed]
    int per_sm[12][kSinkKinds][2] = {};      // resident CTAs per SM (0: not queried yet)
};
std::mutex g_mu;
std::vector<DevInfo> g_dev;

int dev_info(DevInfo **out) {
    int dev;
    CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
    if (!g_dev[dev].sms) {
        CUDA_TRY(cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev));
        CUDA_TRY(cudaDeviceGetAttribute(&g_dev[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    }
    *out = &g_dev[dev];
    return PARBA_OK;
}

template <class Hash, int SINK, bool SEED, bool DEG = false>
int launch_tiles_t(const DevParams &dp, uint64_t lo, uint64_t hi, const SinkArgs &a,
                   unsigned long long *probes, cudaStream_t st, int variant) {
    if (hi <= lo) return PARBA_OK;
    DevInfo *di;
    int rc = dev_info(&di);
    if (rc) return rc;
    auto kern = tile_kernel<Hash, SINK, SEED, DEG>;
    constexpr uint64_t kTile = TileLayout<Hash, SINK>::kTileE;  // this kernel's tile (shadows the default)
    // as many warps per CTA (<= kWarps) as the shared memory allows
    const size_t fixed = TileLayout<Hash, SINK>::fixed, per_warp = TileLayout<Hash, SINK>::per_warp;
    int warps = warps_for(SINK);
    while (warps > 1 && fixed + warps * per_warp > (size_t)di->smem_optin) --warps;
    const size_t smem = fixed + warps * per_warp;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!di->attr_done[variant][SINK][SEED]) {
            const size_t want = fixed + (size_t)warps_for(SINK) * per_warp;
            CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(want > (size_t)di->smem_optin ? di->smem_optin : want)));
            di->attr_done[variant][SINK][SEED] = true;
        }
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        per_sm = di->per_sm[variant][SINK][SEED];
    }
    if (!per_sm) {  // once per kernel and device (a launch of a small chunk should not pay for it)
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem));
        if (per_sm < 1) per_sm = 1;
        std::lock_guard<std::mutex> lk(g_mu);
        di->per_sm[variant][SINK][SEED] = per_sm;
    }
    // launches of at most kLaunchEdgesPerWarp edges per warp (tile-aligned
    // cuts), so the kernel's 32-bit queue cursors never wrap
    const uint64_t max_grid = (uint64_t)di->sms * per_sm;
    const uint64_t cap = max_grid * warps * kLaunchEdgesPerWarp;
    for (uint64_t a0 = lo; a0 < hi;) {
        uint64_t a1 = hi;
        if (hi - a0 > cap) a1 = (a0 / kTile) * kTile + cap;
        const uint64_t tile0 = a0 / kTile;
        const uint64_t ntiles = (a1 - 1) / kTile - tile0 + 1;
        uint64_t grid = max_grid;
        const uint64_t need = (ntiles + warps - 1) / warps;
        if (grid > need) grid = need;
        SinkArgs ac = a;
        if (SINK == kStore) ac.out = a.out + 2 * (a0 - lo);
        if (SINK == kStoreT && !a.hist) ac.t32 = a.t32 + (a0 - lo);
        if (SINK == kStoreT && a.hist) {  // one launch; tile-order slots, every nw-th run per CTA
            if (a1 != hi) return fail(PARBA_ECUDA, "targets pass needs one launch");
            if (ntiles * kTile > a.t32_cap) return fail(PARBA_ECUDA, "targets scratch too small");
            a.t32_geom[0] = ntiles * kTile;
            a.t32_geom[1] = 0;
            a.t32_geom[2] = (uint64_t)warps;
            a.t32_geom[3] = grid;
            a.t32_geom[4] = kTile;
        }
        if (is_targets(SINK)) {  // one launch; every warp owns capw slots
            if (a1 != hi) return fail(PARBA_ECUDA, "targets pass needs one launch");
            const uint64_t nw = grid * warps;
            ac.capw = (ntiles + nw - 1) / nw * kTile;
            if (nw * ac.capw > a.t32_cap) return fail(PARBA_ECUDA, "targets scratch too small");
            a.t32_geom[0] = nw * ac.capw;
            a.t32_geom[1] = ac.capw;
            a.t32_geom[2] = (uint64_t)warps;
            a.t32_geom[3] = grid;
        }
        kern<<<(unsigned)grid, warps * 32, smem, st>>>(dp, a0, a1, tile0, ntiles, ac, probes);
        CUDA_TRY(cudaGetLastError());
        a0 = a1;
    }
    return PARBA_OK;
}

template <class Hash, int SINK>
int launch_tiles_s(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi,
                   const SinkArgs &a, unsigned long long *probes, cudaStream_t st, int variant) {
    if (p->m0 > 0 || p->n0 > 0) return launch_tiles_t<Hash, SINK, true>(dp, lo, hi, a, probes, st, variant);
    return launch_tiles_t<Hash, SINK, false>(dp, lo, hi, a, probes, st, variant);
}

template <int SINK>
int launch_tiles(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi,
                 const SinkArgs &a, unsigned long long *probes, cudaStream_t st) {
    int nc = nc_for(2 * hi - 1);
    if (is_deg(p)) {  // degree sequence: owner lookups instead of closed forms
        if (p->hash_kind == PARBA_HASH_SIMPLE)
            return launch_tiles_t<HashSimple<false>, SINK, true, true>(dp, lo, hi, a, probes, st, 8);
        if (nc <= 3) return launch_tiles_t<HashCrc<3>, SINK, true, true>(dp, lo, hi, a, probes, st, 9);
        if (nc <= 5) return launch_tiles_t<HashCrc<5>, SINK, true, true>(dp, lo, hi, a, probes, st, 10);
        return launch_tiles_t<HashCrc<6>, SINK, true, true>(dp, lo, hi, a, probes, st, 11);
    }
    if (nc <= 3 && p->d >= (1ull << 31)) nc = 4;  // narrow closed forms need d < 2^31
    if (p->hash_kind == PARBA_HASH_SIMPLE) {
        if (nc <= 3) return launch_tiles_s<HashSimple<true>, SINK>(p, dp, lo, hi, a, probes, st, 4);
        return launch_tiles_s<HashSimple<false>, SINK>(p, dp, lo, hi, a, probes, st, 5);
    }
    switch (nc) {
        case 2: return launch_tiles_s<HashCrc<2>, SINK>(p, dp, lo, hi, a, probes, st, 6);
        case 3: return launch_tiles_s<HashCrc<3>, SINK>(p, dp, lo, hi, a, probes, st, 0);
        case 4: return launch_tiles_s<HashCrc<4>, SINK>(p, dp, lo, hi, a, probes, st, 1);
        case 5: return launch_tiles_s<HashCrc<5>, SINK>(p, dp, lo, hi, a, probes, st, 2);
        default: return launch_tiles_s<HashCrc<6>, SINK>(p, dp, lo, hi, a, probes, st, 3);
    }
}

// Targets-only store (kStoreT): CRC families with uniform degree and n <= 2^32
// (callers check; parba_host.cu's host-array path).
int launch_store_targets(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, const SinkArgs &a,
                         unsigned long long *probes, cudaStream_t st) {
    int nc = nc_for(2 * hi - 1);
    if (nc <= 3 && p->d >= (1ull << 31)) nc = 4;
    switch (nc) {
        case 2: return launch_tiles_s<HashCrc<2>, kStoreT>(p, dp, lo, hi, a, probes, st, 6);
        case 3: return launch_tiles_s<HashCrc<3>, kStoreT>(p, dp, lo, hi, a, probes, st, 0);
        case 4: return launch_tiles_s<HashCrc<4>, kStoreT>(p, dp, lo, hi, a, probes, st, 1);
        case 5: return launch_tiles_s<HashCrc<5>, kStoreT>(p, dp, lo, hi, a, probes, st, 2);
        default: return launch_tiles_s<HashCrc<6>, kStoreT>(p, dp, lo, hi, a, probes, st, 3);
    }
}

template <class Hash>
int launch_chains_t(const DevParams &dp, const uint64_t *r0, uint64_t count, uint64_t stop,
                    uint64_t *out, const uint64_t *ids, uint64_t *pairs, unsigned long long *probes,
                    cudaStream_t st) {
    if (dp.W)
        chains_kernel<Hash, true><<<grid_for(count, 256), 256, 0, st>>>(dp, r0, count, stop, out, ids, pairs, probes);
    else
        chains_kernel<Hash><<<grid_for(count, 256), 256, 0, st>>>(dp, r0, count, stop, out, ids, pairs, probes);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int launch_chains(const parba_params_t *p, const DevParams &dp, const uint64_t *r0, uint64_t count,
                  uint64_t stop, uint64_t *out, const uint64_t *ids, uint64_t *pairs,
                  unsigned long long *probes, cudaStream_t st) {
    if (count == 0) return PARBA_OK;
    if (p->hash_kind == PARBA_HASH_SIMPLE)
        return launch_chains_t<HashSimple<false>>(dp, r0, count, stop, out, ids, pairs, probes, st);
    return launch_chains_t<HashCrcBytes>(dp, r0, count, stop, out, ids, pairs, probes, st);
}

template <typename CountT>
int launch_sources(const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K, CountT *counts, cudaStream_t st) {
    // nodes whose edges intersect [lo,hi): v in [src(lo), src(hi-1)] and v >= n0, v < K
    if (hi <= lo) return PARBA_OK;
    if (dp.W) {  // degree sequence: every generated node below K, overlap from W
        const uint64_t vhi = K < dp.n ? K : dp.n;
        if (dp.n0 >= vhi) return PARBA_OK;
        source_counts_kernel<CountT, true><<<grid_for(vhi - dp.n0, 256), 256, 0, st>>>(dp, lo, hi, dp.n0, vhi, counts);
        CUDA_TRY(cudaGetLastError());
        return PARBA_OK;
    }
    const uint64_t vlo = (lo - dp.m0) / dp.d + dp.n0;
    uint64_t vhi = (hi - 1 - dp.m0) / dp.d + dp.n0 + 1;
    if (vhi > K) vhi = K;
    if (vlo >= vhi) return PARBA_OK;
    source_counts_kernel<CountT><<<grid_for(vhi - vlo, 256), 256, 0, st>>>(dp, lo, hi, vlo, vhi, counts);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

}  // namespace

namespace parba {
namespace host {
// The plain store path for [lo, hi) (used by the node path: attempt 0 of
// no_parallel_edges is exactly the plain edge).
int launch_store(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t *out,
                 unsigned long long *probes, cudaStream_t st) {
    SinkArgs a{out, nullptr, nullptr};
    return launch_tiles<kStore>(p, dp, lo, hi, a, probes, st);
}
int launch_store_t32(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint32_t *t32,
                     unsigned long long *probes, cudaStream_t st) {
    SinkArgs a{};
    a.t32 = t32;
    return launch_store_targets(p, dp, lo, hi, a, probes, st);
}
}  // namespace host
}  // namespace parba

namespace {  // partitioned degree counts, defined below the first C block
bool use_partitioned(const parba_params_t *p, uint64_t lo, uint64_t hi, uint64_t K);
template <typename CountT>
int count_partitioned(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                      CountT *counts, unsigned long long *probes, cudaStream_t st, bool by_pos = false,
                      bool *sources_done = nullptr, const Route *route = nullptr);
}  // namespace

extern "C" {

int parba_version(void) { return 20000; }

const char *parba_last_error(void) { return g_err.c_str(); }

int parba_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int parba_hash(const parba_params_t *p, const uint64_t *r, uint64_t count, uint64_t *out, void *stream) {
    int rc = validate(p);
    if (rc) return rc;
    if (count == 0) return PARBA_OK;
    if (!r || !out) return fail(PARBA_EINVAL, "NULL buffer");
    const DevParams dp = make_dev(p);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->hash_kind == PARBA_HASH_SIMPLE)
        hash_kernel<HashSimple<false>><<<grid_for(count, 256), 256, 0, st>>>(dp, r, count, out);
    else
        hash_kernel<HashCrcBytes><<<grid_for(count, 256), 256, 0, st>>>(dp, r, count, out);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

#if PARBA_WARP_TIMES
// diagnostic build only (not in the header): copy the per-warp start/end
// timestamps of the last tile launch.
int parba_debug_warp_times(uint64_t *out, uint64_t nwarps) {
    if (nwarps > kMaxTimedWarps) nwarps = kMaxTimedWarps;
    CUDA_TRY(cudaMemcpyFromSymbol(out, g_warp_times, 2 * nwarps * sizeof(uint64_t)));
    return PARBA_OK;
}
#endif

int parba_crc32c(uint32_t seed, const uint64_t *words, uint64_t count, uint64_t *out, void *stream) {
    if (count == 0) return PARBA_OK;
    if (!words || !out) return fail(PARBA_EINVAL, "NULL buffer");
    crc_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(crc32c_u64_bitwise(seed, 0), words, count,
                                                                      out);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_mulhi_u64(const uint64_t *a, const uint64_t *b, uint64_t count, uint64_t *out, void *stream) {
    if (count == 0) return PARBA_OK;
    if (!a || !b || !out) return fail(PARBA_EINVAL, "NULL buffer");
    mulhi_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(a, b, count, out);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_resolve_chains(const parba_params_t *p, const uint64_t *r0, uint64_t count, uint64_t stop_below,
                         uint64_t *out, unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (rc) return rc;
    if (count == 0) return PARBA_OK;
    if (!r0 || !out) return fail(PARBA_EINVAL, "NULL buffer");
    if (r0 == out) return fail(PARBA_EINVAL, "out may not alias r0");
    return launch_chains(p, make_dev(p), r0, count, stop_below, out, nullptr, nullptr, probes,
                         (cudaStream_t)stream);
}

int parba_generate(const parba_params_t *p, uint64_t lo, uint64_t hi, uint64_t *out_pairs,
                   unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (!rc) rc = check_range(p, lo, hi);
    if (rc) return rc;
    if (hi == lo) return PARBA_OK;
    if (!out_pairs) return fail(PARBA_EINVAL, "out_pairs is NULL");
    if (((uintptr_t)out_pairs) & 15) return fail(PARBA_EINVAL, "out_pairs must be 16-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    const DevParams dp = make_dev(p);
    if (p->flags) {  // node-granular (generator.py:272-302)
        uint64_t vlo, vhi;
        rc = boundary_node(p, dp, lo, &vlo, st);
        if (!rc) rc = boundary_node(p, dp, hi, &vhi, st);
        if (rc) return rc;
        return generate_nodes(p, dp, vlo, vhi, lo, hi, out_pairs, probes, st);
    }
    SinkArgs a{out_pairs, nullptr, nullptr};
    return launch_tiles<kStore>(p, dp, lo, hi, a, probes, st);
}

int parba_generate_targets(const parba_params_t *p, uint64_t lo, uint64_t hi, uint32_t *targets,
                           unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (!rc) rc = check_range(p, lo, hi);
    if (rc) return rc;
    if (!targets_only_ok(p))
        return fail(PARBA_EINVAL, "targets-only store needs the CRC hash, a uniform degree, no option flags "
                                  "and n <= 2^32");
    if (hi == lo) return PARBA_OK;
    if (!targets) return fail(PARBA_EINVAL, "targets is NULL");
    if (((uintptr_t)targets) & 3) return fail(PARBA_EINVAL, "targets must be 4-byte aligned");
    return launch_store_t32(p, make_dev(p), lo, hi, targets, probes, (cudaStream_t)stream);
}

int parba_edges_at(const parba_params_t *p, const uint64_t *ids, uint64_t count, uint64_t *out_pairs,
                   unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (rc) return rc;
    if (count == 0) return PARBA_OK;
    if (!ids || !out_pairs) return fail(PARBA_EINVAL, "NULL buffer");
    if (((uintptr_t)out_pairs) & 15) return fail(PARBA_EINVAL, "out_pairs must be 16-byte aligned");
    if (p->flags)
        return fail(PARBA_EINVAL, "option flags need whole-node processing; use generate_node_edges");
    const DevParams dp = make_dev(p);
    return launch_chains(p, dp, nullptr, count, dp.stop, nullptr, ids, out_pairs, probes, (cudaStream_t)stream);
}

int parba_degree_window(const parba_params_t *p, uint64_t lo, uint64_t hi, uint64_t K,
                        unsigned long long *counts, unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (!rc) rc = check_range(p, lo, hi);
    if (rc) return rc;
    if (hi == lo) return PARBA_OK;
    if (K > 0 && !counts) return fail(PARBA_EINVAL, "counts is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    DevParams dp = make_dev(p, K);
    if (p->flags) return count_nodes_u64(p, dp, lo, hi, K, counts, probes, st);
    if (use_partitioned(p, lo, hi, K)) {  // large windows: partitioned like the full histogram
        bool src_done = false;
        rc = count_partitioned<unsigned long long>(p, dp, lo, hi, K, counts, probes, st, false, &src_done);
        if (rc || src_done) return rc;
        return launch_sources<unsigned long long>(dp, lo, hi, K, counts, st);
    }
    if (is_deg(p)) {
        rc = win_rlim_deg(p, dp, K, st);
        if (rc) return rc;
    }
    SinkArgs a{nullptr, counts, nullptr};
    rc = launch_tiles<kWindow>(p, dp, lo, hi, a, probes, st);
    if (rc) return rc;
    return launch_sources<unsigned long long>(dp, lo, hi, K, counts, st);
}

}  // extern "C"

namespace {

// Partitioned degree counts (parba_hist.cuh) over batches of at most
// kHistBatch edges, for the targets below K (full histogram: K = n, u32
// counts; window: u64 counts).  Applies when targets fit u32 and the domain
// splits into at most kHistBucketsMax buckets of at most 8 slices
// (K <= 8192 * 2^18 = 2^31); more than kHistBuckets buckets are scattered
// in several passes over the batch's targets.  Source endpoints stay
// closed-form (launch_sources).
#ifndef PARBA_HIST_BATCH_LG
#define PARBA_HIST_BATCH_LG 30  // 2^29 -> 2^30: C4 in two batches, [0, 2^30) on the 2-chunk kernel (+1.2%)
#endif
constexpr uint64_t kHistBatch = 1ull << PARBA_HIST_BATCH_LG;
constexpr uint64_t kHistMinEdges = 1ull << 22;
constexpr int kMaxShift = kSliceLg + kMaxSliceLgPerBucket;

// smallest shift with at most kHistBuckets buckets (one scatter pass), capped
// at 8 slices per bucket; 0 when the domain needs more than kHistBucketsMax
int hist_shift(uint64_t K) {
    int shift = kSliceLg;
    while (shift < kMaxShift && ((K + (1ull << shift) - 1) >> shift) > (uint64_t)kHistBuckets) ++shift;
    return ((K + (1ull << shift) - 1) >> shift) <= (uint64_t)kHistBucketsMax ? shift : 0;
}

// PARBA_ONE_SLICE=0: power-of-two bucket widths on the store-targets path too (A/B)
bool one_slice_enabled() {
    const char *e = getenv("PARBA_ONE_SLICE");
    return !(e && e[0] == '0');
}

// PARBA_STT=0: the full histogram's targets pass by the per-step targets
// sink (kTargets) instead of the store-targets sink (A/B)
bool stt_enabled() {
    const char *e = getenv("PARBA_STT");
    return !(e && e[0] == '0');
}

// The position pass (PARBA_POS_MODE=1) measured slower than resolving owners
// in the targets pass (f4 full, n=1e8, m=1.29e9: 2.13e10 vs 3.35e10 edges/s:
// the position domain is 13x the node domain -- 3 scatter passes, 8 slices
// per bucket, and the whole dense map read per batch), so it is opt-in.
// PARBA_FOLD_SOURCES=0: closed-form sources by their own kernel (A/B)
bool fold_enabled() {
    const char *e = getenv("PARBA_FOLD_SOURCES");
    return !(e && e[0] == '0');
}

// PARBA_OFF16=0: one-slice buckets keep u32 targets in the sorted array
// instead of u16 offsets (A/B)
bool off16_enabled() {
    const char *e = getenv("PARBA_OFF16");
    return !(e && e[0] == '0');
}

bool pos_mode_enabled() {
    const char *e = getenv("PARBA_POS_MODE");
    return e && strcmp(e, "1") == 0;
}

bool use_partitioned(const parba_params_t *p, uint64_t lo, uint64_t hi, uint64_t K) {
    // PARBA_FULL_MODE = "direct" / "partition" (tests, A/B)
    const char *e = getenv("PARBA_FULL_MODE");
    const int mode = !e ? 0 : strcmp(e, "direct") == 0 ? 1 : strcmp(e, "partition") == 0 ? 2 : 0;
    if (p->flags || K == 0 || K >= kEmptyTarget) return false;  // targets >= K are never stored
    if (!hist_shift(K)) return false;
    if (mode) return mode == 2;
    // an L2-resident count array (K < 2^25 words) absorbs direct atomics as fast
    return hi - lo >= kHistMinEdges && K >= (1ull << 25);
}

// Scratch of one partitioned count: targets (t32), targets grouped by
// bucket (srt), bucket x column histogram (H) and its exclusive scan (O),
// CUB temp, count work items.
struct PartScratch {
    AsyncBuf t32, srt, H, O, tmp, items;
    size_t tmp_bytes = 0;
    uint64_t stride_nw = 0, stride_ntiles = 0;  // store-targets input: tile-order slots (bucket_scatter_kernel)
    int stride_tlg = 8;                         //   log2 of that launch's tile edges
    uint64_t max_items = 0;
    int shift = 0, nb = 0, spb_lg = 0;
    uint32_t bw = 0;   // bucket width (nodes)
    Magic32 bdiv{};    // bucket = target / bw
    // one_slice: buckets of any width <= kSliceMax, each counted by one CTA
    // (the tile-kernel targets passes; rows input and positions use
    // power-of-two widths)
    int init(uint64_t K, uint64_t slots, uint32_t cols, cudaStream_t st, bool one_slice = false) {
        shift = hist_shift(K);
        nb = (int)((K + (1ull << shift) - 1) >> shift);
        spb_lg = shift - kSliceLg;
        bw = 1u << shift;
        bdiv = Magic32{1u, (uint32_t)shift};
        if (one_slice && spb_lg > 0 && K < (1ull << 31) && (K + kHistBuckets - 1) / kHistBuckets <= kSliceMax) {
            bw = (uint32_t)((K + kHistBuckets - 1) / kHistBuckets);
            nb = (int)((K + bw - 1) / bw);
            spb_lg = 0;
            bdiv = make_magic32(bw);
        }
        max_items = nb + slots / kCountChunk + 1;
        int rc;
        if ((rc = t32.alloc(slots * 4, st)) || (rc = srt.alloc(slots * 4, st)) ||
            (rc = H.alloc((size_t)nb * cols * 4, st)) || (rc = O.alloc((size_t)nb * cols * 4, st)) ||
            (rc = items.alloc((max_items + 1) * 4, st)))
            return rc;
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint32_t *)H.p, (uint32_t *)O.p,
                                               (int64_t)nb * cols, st));
        if ((rc = tmp.alloc(tmp_bytes, st))) return rc;
        std::lock_guard<std::mutex> lk(g_mu);
        static bool attr[64] = {};
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        if (dev < 64 && !attr[dev]) {
            CUDA_TRY(cudaFuncSetAttribute(slice_count_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kSliceMax * 4));
            CUDA_TRY(cudaFuncSetAttribute(slice_count_kernel<unsigned long long>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceMax * 4));
            CUDA_TRY(cudaFuncSetAttribute(slice_count_pos_kernel<uint32_t>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceNodes * 4));
            CUDA_TRY(cudaFuncSetAttribute(bucket_scatter_kernel<kScatterThreads>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kScatterSmem));
            CUDA_TRY(cudaFuncSetAttribute(bucket_scatter_kernel<kScatterThreads, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kScatterSmem));
            CUDA_TRY(cudaFuncSetAttribute(slice_count_kernel<uint32_t, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceMax * 4));
            CUDA_TRY(cudaFuncSetAttribute(slice_count_kernel<unsigned long long, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceMax * 4));
            CUDA_TRY(cudaFuncSetAttribute(slice_count_kernel<uint32_t, false, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceMax * 4));
            CUDA_TRY(cudaFuncSetAttribute(slice_count_kernel<uint32_t, true, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSliceMax * 4));
            attr[dev] = true;
        }
        return PARBA_OK;
    }
    // t32 / H filled for `cols` columns (column c: slots of warps
    // [c / groups * wpc + (c % groups) * wpc / groups, ...) of capw each):
    // scan, scatter passes, plan, slice counts
    // dense != nullptr: the domain is positions [m0, m) of a degree sequence,
    // counted into their owners (slice_count_pos_kernel)
    template <typename CountT>
    int count(uint64_t len, uint64_t capw, uint32_t wpc, uint32_t groups, uint32_t cols, uint64_t K,
              CountT *counts, cudaStream_t st, const uint32_t *dense = nullptr, uint64_t m0 = 0,
              SrcFold fold = SrcFold{}, const Route *route = nullptr) {
        uint32_t *n_items = (uint32_t *)items.p + max_items;
        CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, (const uint32_t *)H.p, (uint32_t *)O.p,
                                               (int64_t)nb * cols, st));
        // one-slice buckets narrower than 2^16 nodes: u16 offsets in the sorted array
        const bool off16 = !dense && spb_lg == 0 && bw <= 0xffffu && off16_enabled();
        for (int wb = 0; wb < nb; wb += kHistBuckets) {  // scatter passes
            const int nbw = nb - wb < kHistBuckets ? nb - wb : kHistBuckets;
            if (off16)
                bucket_scatter_kernel<kScatterThreads, true><<<cols, kScatterThreads, kScatterSmem, st>>>(
                    (const uint32_t *)t32.p, len, wpc, groups, capw, bdiv, wb, nbw, (const uint32_t *)O.p,
                    (uint32_t *)srt.p, stride_nw, stride_ntiles, bw, stride_tlg);
            else
                bucket_scatter_kernel<kScatterThreads><<<cols, kScatterThreads, kScatterSmem, st>>>(
                    (const uint32_t *)t32.p, len, wpc, groups, capw, bdiv, wb, nbw, (const uint32_t *)O.p,
                    (uint32_t *)srt.p, stride_nw, stride_ntiles, 0, stride_tlg);
            CUDA_TRY(cudaGetLastError());
        }
        count_plan_kernel<<<1, kHistThreads, 0, st>>>((const uint32_t *)O.p, (const uint32_t *)H.p, cols, nb,
                                                       (uint32_t *)items.p, n_items, fold.on);
        CUDA_TRY(cudaGetLastError());
        const uint64_t items_ub = nb + len / kCountChunk + 1;  // >= sum of ceil(size_b / chunk)
        if constexpr (sizeof(CountT) == 4) {
            if (route && route->n > 0) {  // counters added straight into their owners' slices
                if (dense) return fail(PARBA_EINVAL, "routed counts do not take the position pass");
                if (off16)
                    slice_count_kernel<CountT, true, true><<<(unsigned)items_ub, kHistThreads, (size_t)bw * 4, st>>>(
                        (const uint32_t *)srt.p, (const uint32_t *)O.p, (const uint32_t *)H.p, cols, nb,
                        (const uint32_t *)items.p, n_items, (uint32_t)K, bw, 0, nullptr, fold, *route);
                else
                    slice_count_kernel<CountT, false, true><<<(unsigned)(items_ub << spb_lg), kHistThreads,
                                                              (spb_lg ? (size_t)kSliceNodes : (size_t)bw) * 4, st>>>(
                        (const uint32_t *)srt.p, (const uint32_t *)O.p, (const uint32_t *)H.p, cols, nb,
                        (const uint32_t *)items.p, n_items, (uint32_t)K, bw, spb_lg, nullptr, fold, *route);
                CUDA_TRY(cudaGetLastError());
                return PARBA_OK;
            }
        }
        if (dense)
            slice_count_pos_kernel<CountT><<<(unsigned)(items_ub << spb_lg), kHistThreads, kSliceNodes * 4, st>>>(
                (const uint32_t *)srt.p, (const uint32_t *)O.p, (const uint32_t *)H.p, cols, nb,
                (const uint32_t *)items.p, n_items, m0, K, shift, spb_lg, dense, counts);
        else if (off16)
            slice_count_kernel<CountT, true><<<(unsigned)items_ub, kHistThreads, (size_t)bw * 4, st>>>(
                (const uint32_t *)srt.p, (const uint32_t *)O.p, (const uint32_t *)H.p, cols, nb,
                (const uint32_t *)items.p, n_items, (uint32_t)K, bw, 0, counts, fold);
        else
            slice_count_kernel<CountT><<<(unsigned)(items_ub << spb_lg), kHistThreads,
                                         (spb_lg ? (size_t)kSliceNodes : (size_t)bw) * 4, st>>>(
                (const uint32_t *)srt.p, (const uint32_t *)O.p, (const uint32_t *)H.p, cols, nb,
                (const uint32_t *)items.p, n_items, (uint32_t)K, bw, spb_lg, counts, fold);
        CUDA_TRY(cudaGetLastError());
        return PARBA_OK;
    }
};

// by_pos (full histogram of a degree sequence with the dense owner map): the
// targets pass emits positions, K becomes the position domain m, and the
// counts are resolved to owners in order.
template <typename CountT>
int count_partitioned(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                      CountT *counts, unsigned long long *probes, cudaStream_t st, bool by_pos,
                      bool *sources_done, const Route *route) {
    if (by_pos) K = p->m;
    // uniform degree: the closed-form sources ride along with the last
    // batch's slice count (no separate pass over the counts)
    const bool fold_src = sources_done && !is_deg(p) && !by_pos && p->d >= 1 && fold_enabled();
    if (sources_done) *sources_done = false;
    DevInfo *di;
    int rc = dev_info(&di);
    if (rc) return rc;
    const uint64_t batch = hi - lo < kHistBatch ? hi - lo : kHistBatch;
    // a launch fills nw * ceil(ntiles / nw) * kTile slots, nw <= 64 warps per SM
    // (tiles of up to 2 * kTile edges: the streaming sinks' 512-edge tiles)
    const uint64_t cap = (batch / kTile + 4) * kTile + (uint64_t)di->sms * 64 * 2 * kTile;
    const uint32_t nblk = (uint32_t)di->sms * 4 * kHistGroups;  // >= warp groups of one tile launch
    PartScratch ps;
    const bool stt = K >= p->n && !by_pos && targets_only_ok(p) && stt_enabled();
    // one-slice buckets (width K/2048, counted by one CTA each) for every
    // tile-kernel targets pass but the position pass (power-of-two slices)
    if ((rc = ps.init(K, cap, nblk, st, !by_pos && one_slice_enabled()))) return rc;
    for (uint64_t b0 = lo; b0 < hi;) {
        uint64_t b1 = hi - b0 > batch ? (b0 / kTile) * kTile + batch : hi;
        if (b1 > hi) b1 = hi;
        uint64_t geom[5] = {};
        SinkArgs a{};
        a.t32 = (uint32_t *)ps.t32.p;
        a.hist = (uint32_t *)ps.H.p;  // the tile launch writes the bucket histogram of each CTA's region
        a.shift = ps.shift;
        a.nb = ps.nb;
        a.bdiv = ps.bdiv;
        a.klim = K;
        if constexpr (sizeof(CountT) == 4) {
            a.by_pos = by_pos ? 1 : 0;
            a.full = (uint32_t *)counts;  // seed-graph targets of the position pass
        }
        a.t32_cap = cap;
        a.t32_geom = geom;
        // the full histogram of a plain CRC family: the store-targets sink
        // (terminal values staged per tile, targets written in tile order with
        // all lanes busy, the bucket histogram counted at the flush)
        ps.stride_nw = ps.stride_ntiles = 0;
        if (stt && ps.nb <= kHistBuckets) {
            rc = launch_store_targets(p, dp, b0, b1, a, probes, st);
            ps.stride_nw = geom[2] * geom[3];                       // warps of the launch
            const uint64_t te = geom[4];                            // its tile (256 or 512 edges)
            ps.stride_tlg = te == 512 ? 9 : 8;
            ps.stride_ntiles = (b1 - 1) / te - b0 / te + 1;         // tiles of the batch
        } else {
            rc = K >= p->n ? launch_tiles<kTargets>(p, dp, b0, b1, a, probes, st)
                           : launch_tiles<kTargetsK>(p, dp, b0, b1, a, probes, st);
        }
        if (rc) return rc;
        const uint32_t used = (uint32_t)geom[3] * kHistGroups;
        if (used > nblk) return fail(PARBA_ECUDA, "targets launch wider than the histogram");
        SrcFold fold{};
        if (fold_src && b1 == hi) fold = SrcFold{lo, hi, p->m0, p->n0, p->d, 1};
        if ((rc = ps.count<CountT>(geom[0], geom[1], (uint32_t)geom[2], kHistGroups, used, K, counts, st,
                                   by_pos ? dp.dense : nullptr, p->m0, fold, route)))
            return rc;
        if (fold.on) *sources_done = true;
        b0 = b1;
    }
    return PARBA_OK;
}

}  // namespace

namespace parba {
namespace host {
// Targets (.y) < K of edge rows already in memory, counted by the partitioned
// pass (sources are the caller's); returns PARBA_EINVAL-free false via *done
// when the pass does not apply (the caller counts directly).
template <typename CountT>
int count_rows_partitioned_t(const ulonglong2 *rows, uint64_t n_rows, uint64_t K, CountT *counts, bool *done,
                             cudaStream_t st) {
    *done = false;
    const char *e = getenv("PARBA_FULL_MODE");
    const int mode = !e ? 0 : strcmp(e, "direct") == 0 ? 1 : strcmp(e, "partition") == 0 ? 2 : 0;
    if (K == 0 || K >= kEmptyTarget || !hist_shift(K) || n_rows == 0) return PARBA_OK;
    if (mode == 1 || (mode == 0 && (K < (1ull << 25) || n_rows < kHistMinEdges))) return PARBA_OK;
    DevInfo *di;
    int rc = dev_info(&di);
    if (rc) return rc;
    const uint32_t cols = (uint32_t)di->sms * 2;
    const uint64_t span = (n_rows + cols - 1) / cols + 255 & ~255ull;  // 256-slot multiple
    PartScratch ps;
    if ((rc = ps.init(K, span * cols, cols, st))) return rc;
    rows_targets_kernel<<<cols, 1024, 0, st>>>(rows, n_rows, span, K, ps.shift, ps.nb, (uint32_t *)ps.t32.p,
                                               (uint32_t *)ps.H.p);
    CUDA_TRY(cudaGetLastError());
    if ((rc = ps.count<CountT>(span * cols, span, 1, 1, cols, K, counts, st))) return rc;
    *done = true;
    return PARBA_OK;
}
int count_rows_partitioned(const ulonglong2 *rows, uint64_t n_rows, uint64_t K, uint32_t *counts, bool *done,
                           cudaStream_t st) {
    return count_rows_partitioned_t<uint32_t>(rows, n_rows, K, counts, done, st);
}
int count_rows_partitioned(const ulonglong2 *rows, uint64_t n_rows, uint64_t K, unsigned long long *counts,
                           bool *done, cudaStream_t st) {
    return count_rows_partitioned_t<unsigned long long>(rows, n_rows, K, counts, done, st);
}
}  // namespace host
}  // namespace parba

extern "C" {

int parba_degree_full(const parba_params_t *p, uint64_t lo, uint64_t hi, uint32_t *counts,
                      unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (!rc) rc = check_range(p, lo, hi);
    if (rc) return rc;
    if (hi == lo) return PARBA_OK;
    if (!counts) return fail(PARBA_EINVAL, "counts is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    const DevParams dp = make_dev(p, p->n);
    if (p->flags) return count_nodes_u32(p, dp, lo, hi, p->n, counts, probes, st);
    // degree sequence with the dense owner map: partition positions instead
    // of owners (no random owner lookups in the targets pass)
    const bool by_pos = is_deg(p) && dp.dense && p->m < (1ull << 31) && pos_mode_enabled();
    bool src_done = false;
    if (by_pos ? use_partitioned(p, lo, hi, p->m) : use_partitioned(p, lo, hi, p->n)) {
        rc = count_partitioned<uint32_t>(p, dp, lo, hi, p->n, counts, probes, st, by_pos, &src_done);
    } else {
        SinkArgs a{nullptr, nullptr, counts};
        rc = launch_tiles<kFull>(p, dp, lo, hi, a, probes, st);
    }
    if (rc || src_done) return rc;
    return launch_sources<uint32_t>(dp, lo, hi, p->n, counts, st);
}

// Routed counts apply where the partitioned pass with folded sources does:
// plain uniform-degree CRC/SIMPLE families (no option flags) with n >= 2^25
// nodes and a shard of at least kHistMinEdges edges.
static bool routed_ok(const parba_params_t *p, uint64_t lo, uint64_t hi) {
    return !is_deg(p) && !p->flags && p->d >= 1 && fold_enabled() && use_partitioned(p, lo, hi, p->n);
}

int parba_degree_full_routed_ok(const parba_params_t *p, uint64_t lo, uint64_t hi) {
    if (validate(p) || check_range(p, lo, hi)) return 0;
    return routed_ok(p, lo, hi) ? 1 : 0;
}

int parba_degree_full_routed(const parba_params_t *p, uint64_t lo, uint64_t hi, int nowners,
                             uint32_t *const *slices, uint64_t slice_nodes, unsigned long long *probes,
                             void *stream) {
    int rc = validate(p);
    if (!rc) rc = check_range(p, lo, hi);
    if (rc) return rc;
    if (nowners < 1 || nowners > kMaxOwners || !slices)
        return fail(PARBA_EINVAL, "routed counts take 1..%d owner slices", kMaxOwners);
    if (slice_nodes == 0 || (slice_nodes & 0xffffu) || slice_nodes >= (1ull << 32) ||
        (unsigned __int128)slice_nodes * (unsigned)nowners < p->n)
        return fail(PARBA_EINVAL, "slice_nodes must be a multiple of 65536 with nowners * slice_nodes >= n");
    for (int g = 0; g < nowners; ++g)
        if (!slices[g] && (uint64_t)g * slice_nodes < p->n) return fail(PARBA_EINVAL, "slice %d is NULL", g);
    if (hi == lo) return PARBA_OK;
    if (!routed_ok(p, lo, hi))
        return fail(PARBA_EINVAL,
                    "routed counts need the partitioned full histogram (uniform degree, no option flags, "
                    "n >= 2^25, a shard of >= 2^22 edges); use parba_degree_full and a reduce");
    Route route{};
    for (int g = 0; g < nowners; ++g) route.ptr[g] = slices[g];
    route.slice = (uint32_t)slice_nodes;
    route.n = nowners;
    const DevParams dp = make_dev(p, p->n);
    bool src_done = false;
    rc = count_partitioned<uint32_t>(p, dp, lo, hi, p->n, nullptr, probes, (cudaStream_t)stream, false, &src_done,
                                     &route);
    if (!rc && !src_done) return fail(PARBA_ECUDA, "routed counts: sources were not folded");
    return rc;
}

int parba_count_ids(const uint64_t *ids, uint64_t count, uint64_t K, unsigned long long *counts, void *stream) {
    if (count == 0 || K == 0) return PARBA_OK;
    if (!ids || !counts) return fail(PARBA_EINVAL, "NULL buffer");
    count_ids_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(ids, count, K, counts);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}


}  // extern "C"

// ---------------------------------------------------------------------------
// Roofline denominators measured in the same run as the kernels they judge
// (bench.py): an INT32 issue peak and a write-only HBM peak.

namespace {

constexpr int kPeakIters = 2048;  // x 8 unrolled x 8 chains x 2 ops

__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t *out, uint32_t seed) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 7u + (uint32_t)k;
    const uint32_t c = 0x9E3779B9u;
    for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                // one LOP3 and one IADD3 per step, emitted as written
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(c), "r"((uint32_t)u));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(c));
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x12345678u) out[0] = s;
}

// 32-byte stores (st.global.v4.b64, sm_100), many CTAs in flight: the
// write-only HBM rate rises with outstanding stores (tools/write_probe.cu:
// 6.1 / 6.9 / 7.2 TB/s with 4 / 8 / 16 CTAs of 512 threads per SM)
__global__ void __launch_bounds__(512) write_peak_kernel(uint64_t *out, uint64_t n32) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += (uint64_t)gridDim.x * blockDim.x)
        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + 4 * i), "l"(i), "l"(i ^ 1ull),
                     "l"(i ^ 2ull), "l"(i ^ 3ull)
                     : "memory");
}

}  // namespace

extern "C" {

int parba_peak_int32(uint32_t *scratch, double *lane_ops, void *stream) {
    if (!scratch || !lane_ops) return fail(PARBA_EINVAL, "NULL buffer");
    DevInfo *di;
    int rc = dev_info(&di);
    if (rc) return rc;
    const unsigned blocks = (unsigned)di->sms * 8, threads = 256;
    int_peak_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(scratch, 1u);
    CUDA_TRY(cudaGetLastError());
    *lane_ops = (double)blocks * threads * kPeakIters * 8.0 * 8.0 * 2.0;
    return PARBA_OK;
}

int parba_peak_write(void *buf, uint64_t bytes, void *stream) {
    if (!buf) return fail(PARBA_EINVAL, "NULL buffer");
    if (((uintptr_t)buf) & 15) return fail(PARBA_EINVAL, "buffer must be 16-byte aligned");
    DevInfo *di;
    int rc = dev_info(&di);
    if (rc) return rc;
    if (((uintptr_t)buf) & 31) return fail(PARBA_EINVAL, "buffer must be 32-byte aligned");
    write_peak_kernel<<<(unsigned)di->sms * 32, 512, 0, (cudaStream_t)stream>>>((uint64_t *)buf, bytes / 32);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

}  // extern "C"
