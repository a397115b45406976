// parba_api.cu -- the C ABI (include/parba_b200.h): validation, template
// dispatch (hash family x CRC width x sink), persistent-grid sizing, and the
// host-buffer entry points.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "../../include/parba_b200.h"
#include "parba_kernels.cuh"
#include "parba_nodes.cuh"

using namespace parba;

namespace {

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

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(PARBA_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));      \
    } while (0)

constexpr uint64_t kMaxEdges = 1ull << 58;  // degreeseq.py:27 (MAX_EDGES)

bool is_deg(const parba_params_t *p) { return p->degree_prefix != nullptr; }

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
        if (!p->rank) return fail(PARBA_EINVAL, "degree sequence without its rank directory");
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

DevParams make_dev(const parba_params_t *p, uint64_t K = 0) {
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
    return d;
}

int bits_of(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

// CRC chunk tables needed to cover every chain value of a launch (r < 2*hi):
// 2 -> r < 2^31 (narrow, 32-bit remainder), 3 -> r < 2^32, 4 -> < 2^43,
// 5 -> < 2^52, 6 -> any.
int nc_for(uint64_t two_hi) {
    const int b = bits_of(two_hi);
    if (b <= 31) return 2;
    if (b <= 32) return 3;
    if (b <= 43) return 4;
    if (b <= 52) return 5;
    return 6;
}

struct DevInfo {
    int sms = 0;
    int smem_optin = 0;  // max dynamic shared memory per block
    bool attr_done[12][3][2] = {};  // [hash variant][sink][seed]
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
    // as many warps per CTA (<= kWarps) as the shared memory allows
    const size_t fixed = TileLayout<Hash, SINK>::fixed, per_warp = TileLayout<Hash, SINK>::per_warp;
    int warps = kWarps;
    while (warps > 1 && fixed + warps * per_warp > (size_t)di->smem_optin) --warps;
    const size_t smem = fixed + warps * per_warp;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!di->attr_done[variant][SINK][SEED]) {
            CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(fixed + kWarps * per_warp > (size_t)di->smem_optin ? di->smem_optin : fixed + kWarps * per_warp)));
            di->attr_done[variant][SINK][SEED] = true;
        }
    }
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem));
    if (per_sm < 1) per_sm = 1;
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
    int nc = nc_for(2 * hi);
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

unsigned grid_for(uint64_t count, int threads) {
    uint64_t g = (count + threads - 1) / threads;
    if (g > 148ull * 32) g = 148ull * 32;
    return (unsigned)(g ? g : 1);
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

// ---------------------------------------------------------------------------
// Degree sequences and option flags (host side of parba_nodes.cuh)

// Stream-ordered scratch, freed on the same stream.
struct AsyncBuf {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    ~AsyncBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    int alloc(size_t bytes, cudaStream_t s) {
        st = s;
        CUDA_TRY(cudaMallocAsync(&p, bytes ? bytes : 8, s));
        return PARBA_OK;
    }
};

int read_u64s(const uint64_t *dptr, uint64_t *out, size_t n, cudaStream_t st) {
    CUDA_TRY(cudaMemcpyAsync(out, dptr, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return PARBA_OK;
}

// Degree sequence: node of position pos (m0 <= pos < m) and its edge span.
int owner_span(const DevParams &dp, uint64_t pos, uint64_t span[3], cudaStream_t st) {
    AsyncBuf b;
    int rc = b.alloc(3 * sizeof(uint64_t), st);
    if (rc) return rc;
    owner_span_kernel<<<1, 32, 0, st>>>(dp, pos, (uint64_t *)b.p);
    CUDA_TRY(cudaGetLastError());
    return read_u64s((const uint64_t *)b.p, span, 3, st);
}

// Window test of a degree sequence: node < K  <=>  r < 2 * W[K - n0].
int win_rlim_deg(const parba_params_t *p, DevParams &dp, uint64_t K, cudaStream_t st) {
    if (K <= p->n0) {
        dp.win_rlim = 0;
    } else if (K >= p->n) {
        dp.win_rlim = 2 * p->m;
    } else {
        uint64_t w;
        int rc = read_u64s(p->degree_prefix + (K - p->n0), &w, 1, st);
        if (rc) return rc;
        dp.win_rlim = 2 * w;
    }
    dp.win_rlim32 = dp.win_rlim > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)dp.win_rlim;
    return PARBA_OK;
}

// Node whose first edge is exactly pos (n when pos == m), else EINVAL
// (_owner_at_boundary / _check_node_boundary, generator.py:231-245).
int boundary_node(const parba_params_t *p, const DevParams &dp, uint64_t pos, uint64_t *v, cudaStream_t st) {
    if (pos == p->m) {
        *v = p->n;
        return PARBA_OK;
    }
    if (!is_deg(p)) {
        if ((pos - p->m0) % p->d)
            return fail(PARBA_EINVAL, "batch boundary %llu is not a node boundary", (unsigned long long)pos);
        *v = p->n0 + (pos - p->m0) / p->d;
        return PARBA_OK;
    }
    uint64_t span[3];
    int rc = owner_span(dp, pos, span, st);
    if (rc) return rc;
    if (span[1] != pos)
        return fail(PARBA_EINVAL, "batch boundary %llu is not a node boundary", (unsigned long long)pos);
    *v = span[0];
    return PARBA_OK;
}

uint64_t node_first_edge(const parba_params_t *p, uint64_t v) { return p->m0 + (v - p->n0) * p->d; }

// no_parallel_edges nodes of degree > kBigDegree: node_big_kernel with a
// per-node hash set in scratch, in chunks of at most kBigScratchWords words.
constexpr uint64_t kBigScratchWords = 1ull << 27;  // 1 GiB per chunk

int generate_big_nodes(const parba_params_t *p, const DevParams &dp, const NodeArgs &na, uint64_t vlo,
                       uint64_t vhi, uint64_t lo, uint64_t hi, uint64_t *out, unsigned long long *probes,
                       unsigned long long *fail_edge, cudaStream_t st) {
    int rc;
    if (!is_deg(p)) {  // uniform degree: every node or none is big
        if (p->d <= kBigDegree) return PARBA_OK;
        const uint64_t per = node_big_words(p->d);
        const uint64_t step = kBigScratchWords / per > 0 ? kBigScratchWords / per : 1;
        for (uint64_t v = vlo; v < vhi; v += step) {
            const uint64_t c = vhi - v < step ? vhi - v : step;
            AsyncBuf scratch;
            if ((rc = scratch.alloc(c * per * 8, st))) return rc;
            node_big_kernel<false><<<grid_for(c, 128), 128, 0, st>>>(dp, na, nullptr, v, c, nullptr, 0, per,
                                                                    (uint64_t *)scratch.p, lo, hi - lo,
                                                                    (ulonglong2 *)out, probes, fail_edge);
            CUDA_TRY(cudaGetLastError());
        }
        return PARBA_OK;
    }
    // degree sequence: list of big nodes (CUB select over node ids), scratch
    // offsets by an exclusive scan, processed in chunks of the list
    const uint64_t nv = vhi - vlo;
    AsyncBuf flags, list, nsel, words, offs, tmp;
    if ((rc = flags.alloc(nv, st)) || (rc = list.alloc(nv * 8, st)) || (rc = nsel.alloc(8, st))) return rc;
    big_flags_kernel<<<grid_for(nv, 256), 256, 0, st>>>(dp, vlo, vhi, kBigDegree, (uint8_t *)flags.p);
    CUDA_TRY(cudaGetLastError());
    cub::CountingInputIterator<uint64_t> ids(vlo);
    size_t tb = 0;
    CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tb, ids, (const uint8_t *)flags.p, (uint64_t *)list.p,
                                        (int64_t *)nsel.p, (int64_t)nv, st));
    if ((rc = tmp.alloc(tb, st))) return rc;
    CUDA_TRY(cub::DeviceSelect::Flagged(tmp.p, tb, ids, (const uint8_t *)flags.p, (uint64_t *)list.p,
                                        (int64_t *)nsel.p, (int64_t)nv, st));
    uint64_t nbig;
    if ((rc = read_u64s((const uint64_t *)nsel.p, &nbig, 1, st))) return rc;
    if (nbig == 0) return PARBA_OK;
    if ((rc = words.alloc(nbig * 8, st)) || (rc = offs.alloc((nbig + 1) * 8, st))) return rc;
    big_words_kernel<<<grid_for(nbig, 256), 256, 0, st>>>(dp, (const uint64_t *)list.p, nbig, (uint64_t *)words.p);
    CUDA_TRY(cudaGetLastError());
    AsyncBuf tmp2;
    tb = 0;
    CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, (const uint64_t *)words.p, (uint64_t *)offs.p + 1,
                                           (int64_t)nbig, st));
    if ((rc = tmp2.alloc(tb, st))) return rc;
    CUDA_TRY(cudaMemsetAsync(offs.p, 0, 8, st));
    CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp2.p, tb, (const uint64_t *)words.p, (uint64_t *)offs.p + 1,
                                           (int64_t)nbig, st));
    std::vector<uint64_t> off(nbig + 1);
    if ((rc = read_u64s((const uint64_t *)offs.p, off.data(), nbig + 1, st))) return rc;
    for (uint64_t k0 = 0; k0 < nbig;) {
        uint64_t k1 = k0 + 1;
        while (k1 < nbig && off[k1 + 1] - off[k0] <= kBigScratchWords) ++k1;
        AsyncBuf scratch;
        if ((rc = scratch.alloc((off[k1] - off[k0]) * 8, st))) return rc;
        node_big_kernel<true><<<grid_for(k1 - k0, 128), 128, 0, st>>>(
            dp, na, (const uint64_t *)list.p + k0, 0, k1 - k0, (const uint64_t *)offs.p + k0, off[k0], 0,
            (uint64_t *)scratch.p, lo, hi - lo, (ulonglong2 *)out, probes, fail_edge);
        CUDA_TRY(cudaGetLastError());
        k0 = k1;
    }
    return PARBA_OK;
}

// Edges of nodes [vlo, vhi) (first edge lo) into out, honouring the flags;
// synchronises st to report an infeasible node (InfeasibleTargetsError).
int generate_nodes(const parba_params_t *p, const DevParams &dp, uint64_t vlo, uint64_t vhi, uint64_t lo,
                   uint64_t hi, uint64_t *out, unsigned long long *probes, cudaStream_t st) {
    if (vhi <= vlo) return PARBA_OK;
    NodeArgs na{};
    na.no_self_loops = (p->flags & PARBA_FLAG_NO_SELF_LOOPS) ? 1u : 0u;
    na.no_parallel_edges = (p->flags & PARBA_FLAG_NO_PARALLEL_EDGES) ? 1u : 0u;
    na.max_attempts = p->max_attempts;
    na.base_seed0 = p->base_seed0;
    na.base_seed1 = p->base_seed1;
    na.base_mult = p->base_mult;
    na.simple = p->hash_kind == PARBA_HASH_SIMPLE ? 1u : 0u;
    AsyncBuf fe;
    int rc = fe.alloc(sizeof(unsigned long long), st);
    if (rc) return rc;
    CUDA_TRY(cudaMemsetAsync(fe.p, 0xFF, sizeof(unsigned long long), st));
    const unsigned grid = grid_for(vhi - vlo, 256);
    const uint64_t big = na.no_parallel_edges ? kBigDegree : UINT64_MAX;
    unsigned long long *fep = (unsigned long long *)fe.p;
    if (is_deg(p))
        node_kernel<true><<<grid, 256, 0, st>>>(dp, na, vlo, vhi, lo, hi - lo, (ulonglong2 *)out, probes, fep, big);
    else
        node_kernel<false><<<grid, 256, 0, st>>>(dp, na, vlo, vhi, lo, hi - lo, (ulonglong2 *)out, probes, fep, big);
    CUDA_TRY(cudaGetLastError());
    if (na.no_parallel_edges) {
        rc = generate_big_nodes(p, dp, na, vlo, vhi, lo, hi, out, probes, fep, st);
        if (rc) return rc;
    }
    uint64_t edge;
    rc = read_u64s((const uint64_t *)fe.p, &edge, 1, st);
    if (rc) return rc;
    if (edge == UINT64_MAX) return PARBA_OK;
    uint64_t v, deg;
    if (is_deg(p)) {
        uint64_t span[3];
        rc = owner_span(dp, edge, span, st);
        if (rc) return rc;
        v = span[0];
        deg = span[2] - span[1];
    } else {
        v = p->n0 + (edge - p->m0) / p->d;
        deg = p->d;
    }
    const uint64_t cap = p->max_attempts ? p->max_attempts : 64 * deg;
    return fail(PARBA_EINFEASIBLE,
                "edge %llu of node %llu: no fresh target in %llu attempts "
                "(distinct-target pool may be smaller than the degree)",
                (unsigned long long)edge, (unsigned long long)v, (unsigned long long)cap);
}

// Degree counts of [lo, hi) with option flags: node-aligned chunks generated
// into scratch, then counted (both endpoints < K).
template <typename CountT>
int count_nodes(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                CountT *counts, unsigned long long *probes, cudaStream_t st) {
    uint64_t vlo, vhi;
    int rc = boundary_node(p, dp, lo, &vlo, st);
    if (!rc) rc = boundary_node(p, dp, hi, &vhi, st);
    if (rc) return rc;
    const uint64_t step = is_deg(p) ? (1ull << 20) : ((1ull << 24) / p->d > 0 ? (1ull << 24) / p->d : 1);
    for (uint64_t v = vlo; v < vhi;) {
        const uint64_t v1 = vhi - v > step ? v + step : vhi;
        uint64_t a, b;
        if (is_deg(p)) {
            uint64_t w[2];
            rc = read_u64s(p->degree_prefix + (v - p->n0), &w[0], 1, st);
            if (!rc) rc = read_u64s(p->degree_prefix + (v1 - p->n0), &w[1], 1, st);
            if (rc) return rc;
            a = w[0];
            b = w[1];
        } else {
            a = node_first_edge(p, v);
            b = node_first_edge(p, v1);
        }
        if (b > a) {
            AsyncBuf scratch;
            rc = scratch.alloc((b - a) * 16, st);
            if (!rc) rc = generate_nodes(p, dp, v, v1, a, b, (uint64_t *)scratch.p, probes, st);
            if (rc) return rc;
            if (K > 0) {
                count_pairs_kernel<CountT><<<grid_for(b - a, 256), 256, 0, st>>>(
                    (const ulonglong2 *)scratch.p, b - a, K, counts);
                CUDA_TRY(cudaGetLastError());
            }
        }
        v = v1;
    }
    return PARBA_OK;
}

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
    if (p->flags) return count_nodes<unsigned long long>(p, dp, lo, hi, K, counts, probes, st);
    if (is_deg(p)) {
        rc = win_rlim_deg(p, dp, K, st);
        if (rc) return rc;
    }
    SinkArgs a{nullptr, counts, nullptr};
    rc = launch_tiles<kWindow>(p, dp, lo, hi, a, probes, st);
    if (rc) return rc;
    return launch_sources<unsigned long long>(dp, lo, hi, K, counts, st);
}

int parba_degree_full(const parba_params_t *p, uint64_t lo, uint64_t hi, uint32_t *counts,
                      unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (!rc) rc = check_range(p, lo, hi);
    if (rc) return rc;
    if (hi == lo) return PARBA_OK;
    if (!counts) return fail(PARBA_EINVAL, "counts is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    const DevParams dp = make_dev(p, p->n);
    if (p->flags) return count_nodes<uint32_t>(p, dp, lo, hi, p->n, counts, probes, st);
    SinkArgs a{nullptr, nullptr, counts};
    rc = launch_tiles<kFull>(p, dp, lo, hi, a, probes, st);
    if (rc) return rc;
    return launch_sources<uint32_t>(dp, lo, hi, p->n, counts, st);
}

int parba_count_ids(const uint64_t *ids, uint64_t count, uint64_t K, unsigned long long *counts, void *stream) {
    if (count == 0 || K == 0) return PARBA_OK;
    if (!ids || !counts) return fail(PARBA_EINVAL, "NULL buffer");
    count_ids_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(ids, count, K, counts);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_count_pairs(const uint64_t *pairs, uint64_t count, uint64_t K, unsigned long long *counts,
                      void *stream) {
    if (count == 0 || K == 0) return PARBA_OK;
    if (!pairs || !counts) return fail(PARBA_EINVAL, "NULL buffer");
    count_pairs_kernel<unsigned long long><<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(
        (const ulonglong2 *)pairs, count, K, counts);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

// ---------------------------------------------------------------------------
// Degree-sequence index (f4).

int parba_degseq_prefix(const uint64_t *degrees, uint64_t count, uint64_t m0, uint64_t *W, void *stream) {
    if (!W) return fail(PARBA_EINVAL, "W is NULL");
    if (count > 0 && !degrees) return fail(PARBA_EINVAL, "degrees is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    if (count > 0) {
        size_t tmp_bytes = 0;
        CUDA_TRY(cub::DeviceScan::ExclusiveScan(nullptr, tmp_bytes, degrees, W, cub::Sum(), (uint64_t)m0,
                                                (int64_t)count, st));
        AsyncBuf tmp;
        int rc = tmp.alloc(tmp_bytes, st);
        if (rc) return rc;
        CUDA_TRY(cub::DeviceScan::ExclusiveScan(tmp.p, tmp_bytes, degrees, W, cub::Sum(), (uint64_t)m0,
                                                (int64_t)count, st));
    }
    degseq_last_kernel<<<1, 32, 0, st>>>(degrees, count, m0, W);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_degseq_rank(const uint64_t *W, uint64_t count, uint64_t m, uint64_t n0, void *rank,
                      uint64_t *owners, uint64_t *n_ones, void *stream) {
    if (!W) return fail(PARBA_EINVAL, "W is NULL");
    if (m >= kMaxEdges) return fail(PARBA_EINVAL, "total edge count %llu exceeds the supported maximum",
                                    (unsigned long long)m);
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t words = (m + 63) / 64;
    if (words == 0) {
        if (n_ones) *n_ones = 0;
        return PARBA_OK;
    }
    if (!rank) return fail(PARBA_EINVAL, "rank is NULL");
    ulonglong2 *rk = (ulonglong2 *)rank;
    CUDA_TRY(cudaMemsetAsync(rk, 0, words * sizeof(ulonglong2), st));
    if (count > 0) {
        rank_mark_kernel<<<grid_for(count, 256), 256, 0, st>>>(W, count, rk);
        CUDA_TRY(cudaGetLastError());
    }
    AsyncBuf cnt, before, tmp;
    int rc = cnt.alloc(words * sizeof(uint64_t), st);
    if (!rc) rc = before.alloc(words * sizeof(uint64_t), st);
    if (rc) return rc;
    rank_popc_kernel<<<grid_for(words, 256), 256, 0, st>>>(rk, words, (uint64_t *)cnt.p);
    CUDA_TRY(cudaGetLastError());
    size_t tmp_bytes = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (const uint64_t *)cnt.p, (uint64_t *)before.p,
                                           (int64_t)words, st));
    rc = tmp.alloc(tmp_bytes, st);
    if (rc) return rc;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, (const uint64_t *)cnt.p, (uint64_t *)before.p,
                                           (int64_t)words, st));
    rank_before_kernel<<<grid_for(words, 256), 256, 0, st>>>(rk, (const uint64_t *)before.p, words);
    CUDA_TRY(cudaGetLastError());
    if (owners && count > 0) {
        owners_kernel<<<grid_for(count, 256), 256, 0, st>>>(W, count, n0, rk, owners);
        CUDA_TRY(cudaGetLastError());
    }
    if (n_ones) {
        uint64_t v[2];
        rc = read_u64s((const uint64_t *)before.p + (words - 1), &v[0], 1, st);
        if (!rc) rc = read_u64s((const uint64_t *)cnt.p + (words - 1), &v[1], 1, st);
        if (rc) return rc;
        *n_ones = v[0] + v[1];
    }
    return PARBA_OK;
}

int parba_degseq_dense(const uint64_t *W, uint64_t count, uint64_t m0, uint64_t n0, uint32_t *dense,
                       void *stream) {
    if (count == 0) return PARBA_OK;
    if (!W || !dense) return fail(PARBA_EINVAL, "NULL buffer");
    if (n0 + count > 0xFFFFFFFFull) return fail(PARBA_EINVAL, "the dense owner map needs n < 2^32");
    dense_fill_kernel<<<grid_for(count * 32, 256), 256, 0, (cudaStream_t)stream>>>(W, count, m0, n0, dense);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_rank1(const void *rank, const uint64_t *es, uint64_t count, uint64_t *out, void *stream) {
    if (count == 0) return PARBA_OK;
    if (!rank || !es || !out) return fail(PARBA_EINVAL, "NULL buffer");
    rank1_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>((const ulonglong2 *)rank, es, count, out);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

int parba_node_of_edges(const parba_params_t *p, const uint64_t *es, uint64_t count, uint64_t *out,
                        uint32_t method, void *stream) {
    int rc = validate(p);
    if (rc) return rc;
    if (method > PARBA_RESOLVE_DEFERRED) return fail(PARBA_EINVAL, "unknown resolution %u", method);
    if (!is_deg(p)) return fail(PARBA_EINVAL, "uniform-degree parameters have no prefix index");
    if (count == 0) return PARBA_OK;
    if (!es || !out) return fail(PARBA_EINVAL, "NULL buffer");
    cudaStream_t st = (cudaStream_t)stream;
    const DevParams dp = make_dev(p);
    const uint64_t n_nodes = p->n - p->n0;
    if (method == PARBA_RESOLVE_RANK) {
        node_of_rank_kernel<<<grid_for(count, 256), 256, 0, st>>>(dp, es, count, out);
    } else if (method == PARBA_RESOLVE_BISECT) {
        node_of_bisect_kernel<<<grid_for(count, 256), 256, 0, st>>>(dp, es, count, n_nodes, out);
    } else {
        AsyncBuf idx, skeys, sidx, tmp;
        rc = idx.alloc(count * 8, st);
        if (!rc) rc = skeys.alloc(count * 8, st);
        if (!rc) rc = sidx.alloc(count * 8, st);
        if (rc) return rc;
        iota_kernel<<<grid_for(count, 256), 256, 0, st>>>((uint64_t *)idx.p, count);
        CUDA_TRY(cudaGetLastError());
        size_t tmp_bytes = 0;
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, es, (uint64_t *)skeys.p,
                                                 (const uint64_t *)idx.p, (uint64_t *)sidx.p, (int64_t)count,
                                                 0, 64, st));
        rc = tmp.alloc(tmp_bytes, st);
        if (rc) return rc;
        CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, es, (uint64_t *)skeys.p,
                                                 (const uint64_t *)idx.p, (uint64_t *)sidx.p, (int64_t)count,
                                                 0, 64, st));
        const uint64_t runs = (count + kMergeRun - 1) / kMergeRun;
        merge_owner_kernel<<<grid_for(runs, 128), 128, 0, st>>>(dp, (const uint64_t *)skeys.p,
                                                                (const uint64_t *)sidx.p, count, n_nodes, out);
    }
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer entry points.

namespace {

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// Upload the host seed array; returns a params copy pointing at device memory.
int upload_seed(const parba_params_t *ph, parba_params_t *pd, DevBuf &seed) {
    *pd = *ph;
    if (ph->m0 > 0) {
        if (!ph->seed_edges) return fail(PARBA_EINVAL, "m0 > 0 but seed_edges is NULL");
        const size_t bytes = 2 * ph->m0 * sizeof(uint64_t);
        CUDA_TRY(cudaMalloc(&seed.p, bytes));
        CUDA_TRY(cudaMemcpy(seed.p, ph->seed_edges, bytes, cudaMemcpyHostToDevice));
        pd->seed_edges = (const uint64_t *)seed.p;
    }
    return PARBA_OK;
}

struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() {
        if (s) cudaStreamDestroy(s);
    }
};
struct EventGuard {
    cudaEvent_t e = nullptr;
    ~EventGuard() {
        if (e) cudaEventDestroy(e);
    }
};

int generate_host_impl(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                       uint64_t *probes_host, int device, float *ms);

}  // namespace

int parba_generate_host(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                        uint64_t *probes_host, int device) {
    return generate_host_impl(ph, lo, hi, out_host, probes_host, device, nullptr);
}

namespace {

// generate_block into host memory on one device; *ms (optional) = device
// time from the first launch to the last copy.
int generate_host_impl(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                       uint64_t *probes_host, int device, float *ms) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (!rc) rc = check_range(ph, lo, hi);
    if (rc) return rc;
    if (probes_host) *probes_host = 0;
    if (ms) *ms = 0.f;
    if (hi == lo) return PARBA_OK;
    if (!out_host) return fail(PARBA_EINVAL, "out_pairs_host is NULL");
    CUDA_TRY(cudaSetDevice(device));
    parba_params_t pd;
    DevBuf seed, bufs, prb;
    rc = upload_seed(ph, &pd, seed);
    if (rc) return rc;
    // Two chunk buffers: the kernel fills one while the other drains over PCIe.
    const uint64_t total = hi - lo;
    uint64_t chunk = total < (1ull << 25) ? total : (1ull << 25);  // 32 Mi edges = 512 MiB
    if (ph->flags && chunk < total) chunk = chunk / ph->d > 0 ? (chunk / ph->d) * ph->d : ph->d;  // node cuts
    const size_t cbytes = chunk * 16;
    CUDA_TRY(cudaMalloc(&bufs.p, 2 * cbytes));
    CUDA_TRY(cudaMalloc(&prb.p, sizeof(unsigned long long)));
    StreamGuard sc, sx;
    CUDA_TRY(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&sx.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaMemsetAsync(prb.p, 0, sizeof(unsigned long long), sc.s));
    EventGuard t0, t1;
    CUDA_TRY(cudaEventCreate(&t0.e));
    CUDA_TRY(cudaEventCreate(&t1.e));
    CUDA_TRY(cudaEventRecord(t0.e, sc.s));
    EventGuard made[2], drained[2];
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(cudaEventCreateWithFlags(&made[b].e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&drained[b].e, cudaEventDisableTiming));
    }
    uint64_t k = 0;
    for (uint64_t a = lo; a < hi; a += chunk, ++k) {
        const uint64_t b = a + chunk < hi ? a + chunk : hi;
        const int slot = (int)(k & 1);
        uint64_t *dbuf = (uint64_t *)((char *)bufs.p + slot * cbytes);
        if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(sc.s, drained[slot].e, 0));
        rc = parba_generate(&pd, a, b, dbuf, (unsigned long long *)prb.p, sc.s);
        if (rc) return rc;
        CUDA_TRY(cudaEventRecord(made[slot].e, sc.s));
        CUDA_TRY(cudaStreamWaitEvent(sx.s, made[slot].e, 0));
        CUDA_TRY(cudaMemcpyAsync(out_host + 2 * (a - lo), dbuf, (b - a) * 16, cudaMemcpyDeviceToHost, sx.s));
        CUDA_TRY(cudaEventRecord(drained[slot].e, sx.s));
    }
    CUDA_TRY(cudaEventRecord(t1.e, sx.s));
    unsigned long long pr = 0;
    CUDA_TRY(cudaStreamSynchronize(sc.s));
    CUDA_TRY(cudaMemcpy(&pr, prb.p, sizeof(pr), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaStreamSynchronize(sx.s));
    if (ms) CUDA_TRY(cudaEventElapsedTime(ms, t0.e, t1.e));
    if (probes_host) *probes_host = pr;
    return PARBA_OK;
}

}  // namespace

int parba_degree_window_host(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t K,
                             int64_t *counts_host, uint64_t *probes_host, int device) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (!rc) rc = check_range(ph, lo, hi);
    if (rc) return rc;
    if (probes_host) *probes_host = 0;
    if (K > 0 && !counts_host) return fail(PARBA_EINVAL, "counts_host is NULL");
    CUDA_TRY(cudaSetDevice(device));
    parba_params_t pd;
    DevBuf seed, cnt, prb;
    rc = upload_seed(ph, &pd, seed);
    if (rc) return rc;
    const size_t cbytes = (K ? K : 1) * sizeof(unsigned long long);
    CUDA_TRY(cudaMalloc(&cnt.p, cbytes));
    CUDA_TRY(cudaMalloc(&prb.p, sizeof(unsigned long long)));
    StreamGuard sc;
    CUDA_TRY(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaMemsetAsync(cnt.p, 0, cbytes, sc.s));
    CUDA_TRY(cudaMemsetAsync(prb.p, 0, sizeof(unsigned long long), sc.s));
    rc = parba_degree_window(&pd, lo, hi, K, (unsigned long long *)cnt.p, (unsigned long long *)prb.p, sc.s);
    if (rc) return rc;
    std::vector<unsigned long long> tmp(K ? K : 1);
    unsigned long long pr = 0;
    CUDA_TRY(cudaMemcpyAsync(tmp.data(), cnt.p, cbytes, cudaMemcpyDeviceToHost, sc.s));
    CUDA_TRY(cudaMemcpyAsync(&pr, prb.p, sizeof(pr), cudaMemcpyDeviceToHost, sc.s));
    CUDA_TRY(cudaStreamSynchronize(sc.s));
    for (uint64_t v = 0; v < K; ++v) counts_host[v] += (int64_t)tmp[v];
    if (probes_host) *probes_host = pr;
    return PARBA_OK;
}

// ---------------------------------------------------------------------------
// Single-process multi-GPU driver (SURVEY.md 8b parba_multi_run): contiguous
// shards on `ndev` devices driven by one host thread each; degree counts are
// summed on devs[0] (peer copies over NVLink + an add kernel) and returned
// once.  torch.distributed / NCCL serve the one-process-per-GPU path
// (paper_1602_07106_b200.parallel); this entry point serves C / FFI callers.

}  // extern "C"

namespace {

template <typename T>
__global__ void add_counts_kernel(T *acc, const T *__restrict__ x, uint64_t n) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
        acc[k] += x[k];
}

struct ShardRun {
    int dev = 0;
    uint64_t a = 0, b = 0;
    int rc = PARBA_OK;
    std::string err;
    uint64_t probes = 0;
    float ms = 0.f;
    void *counts = nullptr;  // device counts of this shard (modes 1, 2)
};

void run_shard(const parba_params_t *ph, int mode, uint64_t K, ShardRun &s, void *out_host) {
    auto done = [&](int rc) {
        s.rc = rc;
        if (rc) s.err = g_err;
    };
    if (mode == PARBA_MULTI_STORE) {
        done(generate_host_impl(ph, s.a, s.b, (uint64_t *)out_host + 2 * (s.a - ph->m0), &s.probes, s.dev, &s.ms));
        return;
    }
    if (cudaSetDevice(s.dev) != cudaSuccess) return done(fail(PARBA_ECUDA, "cudaSetDevice(%d) failed", s.dev));
    parba_params_t pd;
    DevBuf seed, prb;
    int rc = upload_seed(ph, &pd, seed);
    if (rc) return done(rc);
    StreamGuard st;
    EventGuard t0, t1;
    if (cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking) != cudaSuccess || cudaEventCreate(&t0.e) ||
        cudaEventCreate(&t1.e) || cudaMalloc(&prb.p, 8) || cudaMemsetAsync(prb.p, 0, 8, st.s))
        return done(fail(PARBA_ECUDA, "shard setup on device %d failed", s.dev));
    const size_t bytes = mode == PARBA_MULTI_FULL ? (size_t)ph->n * 4 : (size_t)(K ? K : 1) * 8;
    if (mode != PARBA_MULTI_DISCARD) {
        if (cudaMalloc(&s.counts, bytes) || cudaMemsetAsync(s.counts, 0, bytes, st.s))
            return done(fail(PARBA_ENOMEM, "count buffer of %zu bytes on device %d", bytes, s.dev));
    }
    cudaEventRecord(t0.e, st.s);
    if (mode == PARBA_MULTI_FULL)
        rc = parba_degree_full(&pd, s.a, s.b, (uint32_t *)s.counts, (unsigned long long *)prb.p, st.s);
    else
        rc = parba_degree_window(&pd, s.a, s.b, mode == PARBA_MULTI_DISCARD ? 0 : K,
                                 (unsigned long long *)s.counts, (unsigned long long *)prb.p, st.s);
    if (rc) return done(rc);
    cudaEventRecord(t1.e, st.s);
    unsigned long long pr = 0;
    if (cudaMemcpyAsync(&pr, prb.p, 8, cudaMemcpyDeviceToHost, st.s) || cudaStreamSynchronize(st.s) ||
        cudaEventElapsedTime(&s.ms, t0.e, t1.e))
        return done(fail(PARBA_ECUDA, "shard on device %d: %s", s.dev, cudaGetErrorString(cudaGetLastError())));
    s.probes = pr;
    done(PARBA_OK);
}

// Sum the shards' device counts on devs[0] and add them into the host array.
template <typename T>
int reduce_shards(std::vector<ShardRun> &sh, uint64_t n, int64_t *out_host, float *ms) {
    const int d0 = sh[0].dev;
    CUDA_TRY(cudaSetDevice(d0));
    StreamGuard st;
    EventGuard t0, t1;
    CUDA_TRY(cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreate(&t0.e));
    CUDA_TRY(cudaEventCreate(&t1.e));
    CUDA_TRY(cudaEventRecord(t0.e, st.s));
    DevBuf stage;
    if (sh.size() > 1) CUDA_TRY(cudaMalloc(&stage.p, n * sizeof(T)));
    for (size_t g = 1; g < sh.size(); ++g) {
        CUDA_TRY(cudaMemcpyPeerAsync(stage.p, d0, sh[g].counts, sh[g].dev, n * sizeof(T), st.s));
        add_counts_kernel<T><<<grid_for(n, 256), 256, 0, st.s>>>((T *)sh[0].counts, (const T *)stage.p, n);
        CUDA_TRY(cudaGetLastError());
    }
    std::vector<T> tmp(n);
    CUDA_TRY(cudaMemcpyAsync(tmp.data(), sh[0].counts, n * sizeof(T), cudaMemcpyDeviceToHost, st.s));
    CUDA_TRY(cudaEventRecord(t1.e, st.s));
    CUDA_TRY(cudaStreamSynchronize(st.s));
    CUDA_TRY(cudaEventElapsedTime(ms, t0.e, t1.e));
    for (uint64_t v = 0; v < n; ++v) out_host[v] += (int64_t)tmp[v];
    return PARBA_OK;
}

}  // namespace

extern "C" {

int parba_multi_run(const parba_params_t *ph, int ndev, const int *devs, int mode, uint64_t K, void *out_host,
                    uint64_t *probes_host, double *device_seconds) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (rc) return rc;
    if (ndev < 1 || !devs) return fail(PARBA_EINVAL, "need ndev >= 1 devices");
    if (mode < PARBA_MULTI_STORE || mode > PARBA_MULTI_DISCARD) return fail(PARBA_EINVAL, "unknown mode %d", mode);
    if (mode == PARBA_MULTI_FULL) K = ph->n;
    if (!out_host && (mode == PARBA_MULTI_STORE || ((mode == PARBA_MULTI_WINDOW || mode == PARBA_MULTI_FULL) && K)))
        return fail(PARBA_EINVAL, "out_host is NULL");
    if (mode == PARBA_MULTI_FULL && 2 * (unsigned __int128)ph->m >= ((unsigned __int128)1 << 32))
        return fail(PARBA_EINVAL, "full histogram needs 2m < 2^32 (uint32 counters); use the window mode");
    const uint64_t total = ph->m - ph->m0;
    std::vector<ShardRun> sh(ndev);
    for (int g = 0; g < ndev; ++g) {
        sh[g].dev = devs[g];
        sh[g].a = ph->m0 + (uint64_t)(((unsigned __int128)total * g) / ndev);
        sh[g].b = ph->m0 + (uint64_t)(((unsigned __int128)total * (g + 1)) / ndev);
        if (ph->flags) {  // node-granular: cut at node boundaries (uniform d)
            if (g > 0) sh[g].a = node_first_edge(ph, ph->n0 + (sh[g].a - ph->m0) / ph->d);
            if (g < ndev - 1) sh[g].b = node_first_edge(ph, ph->n0 + (sh[g].b - ph->m0) / ph->d);
        }
    }
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) th.emplace_back(run_shard, ph, mode, K, std::ref(sh[g]), out_host);
    for (auto &t : th) t.join();
    rc = PARBA_OK;
    std::string err;
    uint64_t probes = 0;
    float worst = 0.f;
    for (auto &s : sh) {
        if (s.rc && !rc) {
            rc = s.rc;
            err = s.err;
        }
        probes += s.probes;
        worst = s.ms > worst ? s.ms : worst;
    }
    float red_ms = 0.f;
    if (!rc && mode == PARBA_MULTI_WINDOW && K)
        rc = reduce_shards<unsigned long long>(sh, K, (int64_t *)out_host, &red_ms);
    else if (!rc && mode == PARBA_MULTI_FULL)
        rc = reduce_shards<uint32_t>(sh, K, (int64_t *)out_host, &red_ms);
    for (auto &s : sh)
        if (s.counts) {
            cudaSetDevice(s.dev);
            cudaFree(s.counts);
        }
    if (rc) return err.empty() ? rc : fail(rc, "%s", err.c_str());
    if (probes_host) *probes_host = probes;
    if (device_seconds) *device_seconds = (worst + red_ms) / 1000.0;
    return PARBA_OK;
}

}  // extern "C"
