// host_probe.cu -- host-side bandwidth probe for the end-to-end path
// (generate_block into a host array).  Build:
//   nvcc -O3 -std=c++17 -Xcompiler -fopenmp,-O3 -o tools/host_probe tools/host_probe.cu
// Prints one JSON object:
//   d2h_gbs          pinned device->host copy of 4 GiB (cudaMemcpyAsync)
//   fill[t]          host expansion of u32 targets (pinned) into u64 (src,tgt)
//                    rows (pinned, pre-faulted), t threads, NT vs regular stores
//   fill_during_d2h  the same fill while a D2H copy runs (contention)
//   memset[t]        plain streaming-store bandwidth, t threads
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                           \
        }                                                                       \
    } while (0)

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// rows[k] = (lo+k)/d, tgt[k]; NT: 16-byte streaming stores
static void fill_part(uint64_t *rows, const uint32_t *tgt, uint64_t lo, uint64_t a, uint64_t b, uint64_t d, bool nt) {
    uint64_t i = lo + a;
    uint64_t src = i / d, rem = i % d;
    for (uint64_t k = a; k < b; ++k) {
        if (nt) {
            _mm_stream_si128((__m128i *)(rows + 2 * k), _mm_set_epi64x((long long)tgt[k], (long long)src));
        } else {
            rows[2 * k] = src;
            rows[2 * k + 1] = tgt[k];
        }
        if (++rem == d) {
            rem = 0;
            ++src;
        }
    }
    if (nt) _mm_sfence();
}

static double fill(uint64_t *rows, const uint32_t *tgt, uint64_t n, int threads, bool nt) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) {
        uint64_t a = n * t / threads, b = n * (t + 1) / threads;
        a &= ~(uint64_t)7;
        if (t == threads - 1) b = n; else b &= ~(uint64_t)7;
        th.emplace_back(fill_part, rows, tgt, 1000000000ull - n, a, b, 10ull, nt);
    }
    for (auto &x : th) x.join();
    return now() - t0;
}

static void set_part(uint64_t *p, uint64_t a, uint64_t b) {
    __m128i z = _mm_set1_epi64x(0x0102030405060708ll);
    for (uint64_t k = a; k < b; k += 2) _mm_stream_si128((__m128i *)(p + k), z);
    _mm_sfence();
}

static double memset_t(uint64_t *p, uint64_t words, int threads) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) {
        uint64_t a = (words * t / threads) & ~1ull, b = t == threads - 1 ? words : (words * (t + 1) / threads) & ~1ull;
        th.emplace_back(set_part, p, a, b);
    }
    for (auto &x : th) x.join();
    return now() - t0;
}

int main() {
    const uint64_t N = 250000000ull;  // edges per e2e step (bench.py E2E_EDGES)
    unsigned hw = std::thread::hardware_concurrency();
    uint32_t *tgt_h;
    uint64_t *rows_h;
    CK(cudaHostAlloc(&tgt_h, N * 4, 0));
    CK(cudaHostAlloc(&rows_h, N * 16, 0));
    memset(tgt_h, 1, N * 4);
    memset(rows_h, 0, N * 16);
    void *dbuf;
    CK(cudaMalloc(&dbuf, N * 16));
    CK(cudaMemset(dbuf, 3, N * 16));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"hw_threads\": %u", hw);
    // D2H of 4 GB pinned
    float best = 1e9f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, s);
        CK(cudaMemcpyAsync(rows_h, dbuf, N * 16, cudaMemcpyDeviceToHost, s));
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    printf(", \"d2h_gbs\": %.2f", N * 16 / (best * 1e-3) / 1e9);
    best = 1e9f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, s);
        CK(cudaMemcpyAsync(tgt_h, dbuf, N * 4, cudaMemcpyDeviceToHost, s));
        cudaEventRecord(e1, s);
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    printf(", \"d2h_1gb_gbs\": %.2f", N * 4 / (best * 1e-3) / 1e9);
    int tl[] = {1, 2, 4, 8, 12, 16, 24, 32, 48, 64};
    for (int nt = 1; nt >= 0; --nt) {
        printf(", \"fill_%s_edges_per_s\": {", nt ? "nt" : "reg");
        bool first = true;
        for (int t : tl) {
            if ((unsigned)t > hw) break;
            double b = 1e9;
            for (int r = 0; r < 2; ++r) b = std::min(b, fill(rows_h, tgt_h, N, t, nt));
            printf("%s\"%d\": %.4g", first ? "" : ", ", t, N / b);
            first = false;
        }
        printf("}");
    }
    printf(", \"memset_nt_gbs\": {");
    bool first = true;
    for (int t : tl) {
        if ((unsigned)t > hw) break;
        double b = 1e9;
        for (int r = 0; r < 2; ++r) b = std::min(b, memset_t(rows_h, 2 * N, t));
        printf("%s\"%d\": %.2f", first ? "" : ", ", t, N * 16 / b / 1e9);
        first = false;
    }
    printf("}");
    // fill with all threads while a 4 GB D2H (into a separate pinned buffer) runs
    uint64_t *other;
    CK(cudaHostAlloc(&other, N * 16, 0));
    memset(other, 0, N * 16);
    cudaEventRecord(e0, s);
    CK(cudaMemcpyAsync(other, dbuf, N * 16, cudaMemcpyDeviceToHost, s));
    cudaEventRecord(e1, s);
    double fdt = fill(rows_h, tgt_h, N, (int)hw, true);
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"fill_during_d2h\": {\"fill_edges_per_s\": %.4g, \"d2h_gbs\": %.2f}", N / fdt, N * 16 / (ms * 1e-3) / 1e9);
    // pageable (fresh, unfaulted) destination: first-touch cost
    double t0 = now();
    uint64_t *page = (uint64_t *)malloc(N * 16);
    fill(page, tgt_h, N, (int)hw, true);
    printf(", \"fill_fresh_pageable_edges_per_s\": %.4g", N / (now() - t0));
    t0 = now();
    fill(page, tgt_h, N, (int)hw, true);
    printf(", \"fill_faulted_pageable_edges_per_s\": %.4g", N / (now() - t0));
    free(page);
    printf("}\n");
    return 0;
}
