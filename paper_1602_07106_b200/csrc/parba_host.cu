// parba_host.cu -- host-buffer entry points of the C ABI (blocking; the
// device generates in chunks while earlier chunks stream back) and the
// single-process multi-GPU driver parba_multi_run.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/parba_b200.h"
#include "parba_common.h"

using namespace parba;
using namespace parba::host;

extern "C" {

// ---------------------------------------------------------------------------
// Host-buffer entry points.

namespace {

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
