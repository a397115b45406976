// parba_common.h -- host-side internals shared by the C-ABI translation
// units (parba_api.cu, parba_nodes_api.cu, parba_host.cu): error reporting,
// parameter validation, DevParams construction, scratch helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/parba_b200.h"
#include "parba_device.cuh"

namespace parba {
namespace host {

extern thread_local std::string g_err;
int fail(int code, const char *fmt, ...);

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return ::parba::host::fail(PARBA_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

constexpr uint64_t kMaxEdges = 1ull << 58;  // degreeseq.py:27 (MAX_EDGES)

inline bool is_deg(const parba_params_t *p) { return p->degree_prefix != nullptr; }
// First edge of node v of a uniform-degree family.
inline uint64_t node_first_edge(const parba_params_t *p, uint64_t v) { return p->m0 + (v - p->n0) * p->d; }
int validate(const parba_params_t *p);
int check_range(const parba_params_t *p, uint64_t lo, uint64_t hi);
DevParams make_dev(const parba_params_t *p, uint64_t K = 0);

inline unsigned grid_for(uint64_t count, int threads) {
    uint64_t g = (count + threads - 1) / threads;
    if (g > 148ull * 32) g = 148ull * 32;
    return (unsigned)(g ? g : 1);
}

// Keep memory freed by cudaFreeAsync in the device's default pool instead of
// returning it to the driver at every synchronisation (the node paths
// allocate and free GB-sized scratch per call; re-mapping it cost more than
// the kernels).  Idempotent, once per device.
inline void retain_async_pool() {
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[dev] = true;
}

// Stream-ordered scratch, freed on the same stream.
struct AsyncBuf {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    ~AsyncBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    int alloc(size_t bytes, cudaStream_t s) {
        st = s;
        retain_async_pool();
        CUDA_TRY(cudaMallocAsync(&p, bytes ? bytes : 8, s));
        return PARBA_OK;
    }
};
struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};
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

int read_u64s(const uint64_t *dptr, uint64_t *out, size_t n, cudaStream_t st);

int launch_store(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t *out,
                 unsigned long long *probes, cudaStream_t st);

// Targets-only store (the u32 target of each edge in edge order): CRC,
// uniform degree, no option flags, n <= 2^32 (see targets_only_ok).
int launch_store_t32(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint32_t *t32,
                     unsigned long long *probes, cudaStream_t st);
inline bool targets_only_ok(const parba_params_t *p) {
    return !is_deg(p) && !p->flags && p->hash_kind == PARBA_HASH_CRC && p->n <= (1ull << 32);
}

// Node-granular paths (parba_nodes_api.cu): option flags and degree sequences.
int win_rlim_deg(const parba_params_t *p, DevParams &dp, uint64_t K, cudaStream_t st);
int boundary_node(const parba_params_t *p, const DevParams &dp, uint64_t pos, uint64_t *v, cudaStream_t st);
int count_rows_partitioned(const ulonglong2 *rows, uint64_t n_rows, uint64_t K, uint32_t *counts, bool *done,
                           cudaStream_t st);
int count_rows_partitioned(const ulonglong2 *rows, uint64_t n_rows, uint64_t K, unsigned long long *counts,
                           bool *done, cudaStream_t st);
int generate_nodes(const parba_params_t *p, const DevParams &dp, uint64_t vlo, uint64_t vhi, uint64_t lo,
                   uint64_t hi, uint64_t *out, unsigned long long *probes, cudaStream_t st,
                   unsigned long long *fail_ext = nullptr);
int count_nodes_u64(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                    unsigned long long *counts, unsigned long long *probes, cudaStream_t st);
int count_nodes_u32(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                    uint32_t *counts, unsigned long long *probes, cudaStream_t st);

}  // namespace host
}  // namespace parba
