// parba_api.cu -- the C ABI (include/parba_b200.h): validation, template
// dispatch (hash family x CRC width x sink), persistent-grid sizing, and the
// host-buffer entry points.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/parba_b200.h"
#include "parba_kernels.cuh"

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

int validate(const parba_params_t *p) {
    if (!p) return fail(PARBA_EINVAL, "params is NULL");
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
    d.div64 = make_magic64(p->d);
    d.div32 = make_magic32(p->d);
    d.div32_2d = make_magic32(2 * p->d);
    d.K = K;
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
    bool attr_done[8][3][2] = {};  // [hash variant][sink][seed]
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

template <class Hash, int SINK, bool SEED>
int launch_tiles_t(const DevParams &dp, uint64_t lo, uint64_t hi, const SinkArgs &a,
                   unsigned long long *probes, cudaStream_t st, int variant) {
    if (hi <= lo) return PARBA_OK;
    DevInfo *di;
    int rc = dev_info(&di);
    if (rc) return rc;
    auto kern = tile_kernel<Hash, SINK, SEED>;
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
    const uint64_t vlo = (lo - dp.m0) / dp.d + dp.n0;
    uint64_t vhi = (hi - 1 - dp.m0) / dp.d + dp.n0 + 1;
    if (vhi > K) vhi = K;
    if (vlo >= vhi) return PARBA_OK;
    source_counts_kernel<CountT><<<grid_for(vhi - vlo, 256), 256, 0, st>>>(dp, lo, hi, vlo, vhi, counts);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

}  // namespace

extern "C" {

int parba_version(void) { return 10000; }

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
    SinkArgs a{out_pairs, nullptr, nullptr};
    return launch_tiles<kStore>(p, make_dev(p), lo, hi, a, probes, (cudaStream_t)stream);
}

int parba_edges_at(const parba_params_t *p, const uint64_t *ids, uint64_t count, uint64_t *out_pairs,
                   unsigned long long *probes, void *stream) {
    int rc = validate(p);
    if (rc) return rc;
    if (count == 0) return PARBA_OK;
    if (!ids || !out_pairs) return fail(PARBA_EINVAL, "NULL buffer");
    if (((uintptr_t)out_pairs) & 15) return fail(PARBA_EINVAL, "out_pairs must be 16-byte aligned");
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
    const DevParams dp = make_dev(p, K);
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

}  // namespace

int parba_generate_host(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                        uint64_t *probes_host, int device) {
    int rc = validate(ph);
    if (!rc) rc = check_range(ph, lo, hi);
    if (rc) return rc;
    if (probes_host) *probes_host = 0;
    if (hi == lo) return PARBA_OK;
    if (!out_host) return fail(PARBA_EINVAL, "out_pairs_host is NULL");
    CUDA_TRY(cudaSetDevice(device));
    parba_params_t pd;
    DevBuf seed, bufs, prb;
    rc = upload_seed(ph, &pd, seed);
    if (rc) return rc;
    // Two chunk buffers: the kernel fills one while the other drains over PCIe.
    const uint64_t total = hi - lo;
    const uint64_t chunk = total < (1ull << 25) ? total : (1ull << 25);  // 32 Mi edges = 512 MiB
    const size_t cbytes = chunk * 16;
    CUDA_TRY(cudaMalloc(&bufs.p, 2 * cbytes));
    CUDA_TRY(cudaMalloc(&prb.p, sizeof(unsigned long long)));
    StreamGuard sc, sx;
    CUDA_TRY(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&sx.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaMemsetAsync(prb.p, 0, sizeof(unsigned long long), sc.s));
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
    unsigned long long pr = 0;
    CUDA_TRY(cudaStreamSynchronize(sc.s));
    CUDA_TRY(cudaMemcpy(&pr, prb.p, sizeof(pr), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaStreamSynchronize(sx.s));
    if (probes_host) *probes_host = pr;
    return PARBA_OK;
}

int parba_degree_window_host(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t K,
                             int64_t *counts_host, uint64_t *probes_host, int device) {
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

}  // extern "C"
