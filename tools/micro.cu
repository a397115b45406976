// micro.cu -- B200 microbenchmarks for the roofline denominators and the
// per-probe building blocks.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -o tools/micro tools/micro.cu ; run: tools/micro
//
//   int_peak     INT32 lane-ops/s (LOP3/IADD3 mix, 8 independent chains)
//   fp64_peak    DFMA/s
//   write_peak   write-only HBM bandwidth (16-byte streaming stores)
//   mod_*        h % r throughput: fp64-reciprocal path vs the compiler's u64 %
//   crc5         byte-table CRC of a 35-bit word (5 smem lookups)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "../paper_1602_07106_b200/csrc/parba_device.cuh"

using namespace parba;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                        \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int ITERS = 4096;

__global__ void int_peak(uint32_t *out, uint32_t seed) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 7 + k;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[k] = (a[k] ^ (a[k] + 0x9E3779B9u)) + (uint32_t)i;  // LOP3+IADD3 per step after folding
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x12345678u) out[0] = s;
}

__global__ void fp64_peak(double *out, double seed) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x + k;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999, 1e-7);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1.2345) out[0] = s;
}

__global__ void write_peak(ulonglong2 *out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(out + i, make_ulonglong2(i, i ^ 0x5555));
}

// max relative error of rcp.approx.ftz.f64 (no Newton) over r = seed-derived values
__global__ void rcp_err(unsigned long long *worst_bits, uint64_t seed) {
    uint64_t x = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
    double worst = 0;
    for (int k = 0; k < 256; ++k) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const int sh = (int)(x & 63);
        const uint64_t r = (x >> sh) | 1;
        const double rd = (double)r;
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(rd));
        const double e = fabs(fma(-rd, y, 1.0));
        worst = e > worst ? e : worst;
    }
    atomicMax(worst_bits, (unsigned long long)__double_as_longlong(worst));
}

template <int MODE>
__global__ void mod_bench(const uint64_t *__restrict__ r, uint64_t *out, int n, int reps) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t rr = r[i];
    uint32_t hhi = (uint32_t)(rr * 0x9E3779B97F4A7C15ull >> 32), hlo = (uint32_t)rr;
    uint64_t acc = 0;
    for (int k = 0; k < reps; ++k) {
        uint64_t v;
        if (MODE == 0) v = mod_u32r(hhi, hlo, (uint32_t)rr);
        else v = (((uint64_t)hhi << 32) | hlo) % rr;
        acc += v;
        hhi ^= (uint32_t)v;
        hlo += 0x3779B9u;
    }
    out[i] = acc;
}

__global__ void crc_bench(const uint64_t *__restrict__ r, uint64_t *out, int n, int reps) {
    __shared__ CrcTables<5> tabs;
    build_crc_tables<5>(tabs);
    __syncthreads();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t w = r[i];
    uint32_t acc = 0;
    for (int k = 0; k < reps; ++k) {
        acc ^= crc0<5>(tabs, w);
        w = (w + acc) & ((1ull << 35) - 1);
    }
    out[i] = acc;
}

static float time_it(void (*launch)(void *), void *arg, int reps = 5) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch(arg);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int k = 0; k < reps; ++k) {
        CK(cudaEventRecord(a));
        launch(arg);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    return best;
}

struct Ctx {
    int sms;
    void *buf;
    size_t n;
    uint64_t *r, *o;
    int nr, reps;
};

int main() {
    Ctx c{};
    CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, 0));
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = c.sms * 8, threads = 256;
    CK(cudaMalloc(&c.buf, 8ull << 30));
    // INT32
    float ms = time_it([](void *p) { int_peak<<<((Ctx *)p)->sms * 8, 256>>>((uint32_t *)((Ctx *)p)->buf, 1); }, &c);
    // SASS of the unrolled body: 116 INT instructions (IADD3/VIADD/LOP3) per 32 steps
    double int_ops = (double)blocks * threads * ITERS * 8 * (116.0 / 32.0);
    // FP64
    float ms64 = time_it([](void *p) { fp64_peak<<<((Ctx *)p)->sms * 8, 256>>>((double *)((Ctx *)p)->buf, 1.0); }, &c);
    double dfma = (double)blocks * threads * ITERS * 8;
    // write-only HBM
    c.n = (8ull << 30) / 16;
    float msw = time_it([](void *p) {
        Ctx *q = (Ctx *)p;
        write_peak<<<q->sms * 8, 512>>>((ulonglong2 *)q->buf, q->n);
    }, &c);
    // mod / crc
    c.nr = 1 << 22;
    c.reps = 64;
    CK(cudaMalloc(&c.r, c.nr * 8ull));
    CK(cudaMalloc(&c.o, c.nr * 8ull));
    uint64_t *h = (uint64_t *)malloc(c.nr * 8ull);
    srand(1);
    for (int i = 0; i < c.nr; ++i) h[i] = (((uint64_t)rand() << 31) ^ rand()) % (1ull << 31) + 1;
    CK(cudaMemcpy(c.r, h, c.nr * 8ull, cudaMemcpyHostToDevice));
    float msm0 = time_it([](void *p) { Ctx *q = (Ctx *)p; mod_bench<0><<<q->nr / 256, 256>>>(q->r, q->o, q->nr, q->reps); }, &c);
    float msm1 = time_it([](void *p) { Ctx *q = (Ctx *)p; mod_bench<1><<<q->nr / 256, 256>>>(q->r, q->o, q->nr, q->reps); }, &c);
    float msc = time_it([](void *p) { Ctx *q = (Ctx *)p; crc_bench<<<q->nr / 256, 256>>>(q->r, q->o, q->nr, q->reps); }, &c);
    double ops = (double)c.nr * c.reps;
    unsigned long long *wb;
    CK(cudaMalloc(&wb, 8));
    CK(cudaMemset(wb, 0, 8));
    rcp_err<<<c.sms * 32, 256>>>(wb, 12345);
    unsigned long long wbits = 0;
    CK(cudaMemcpy(&wbits, wb, 8, cudaMemcpyDeviceToHost));
    double werr;
    memcpy(&werr, &wbits, 8);
    printf("{\"rcp_approx_f64_max_rel_err\": %.3e, \"log2\": %.2f}\n", werr, log2(werr));
    printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"int32_lane_ops_per_s\": %.4e, \"dfma_per_s\": %.4e, "
           "\"write_only_gbs\": %.1f, \"mod_fp64_per_s\": %.4e, \"mod_u64_percent_per_s\": %.4e, "
           "\"crc5_per_s\": %.4e}\n",
           c.sms, clk_khz, int_ops / (ms * 1e-3), dfma / (ms64 * 1e-3), (8ull << 30) / (msw * 1e-3) / 1e9,
           ops / (msm0 * 1e-3), ops / (msm1 * 1e-3), ops / (msc * 1e-3));
    return 0;
}
