// atomic_probe.cu -- L2 atomic throughput for the C4 full-histogram design
// question: can a counts slice that fits in L2 absorb one RED.ADD.U32 per
// target fast enough that P passes over a u32 target stream (each pass
// counting only the targets of one node slice) beat the bucket sort?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/atomic_probe tools/atomic_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));           \
            return 1;                                                          \
        }                                                                      \
    } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// targets with the BA skew: v = floor(n * u^2) has density ~ 1/sqrt(v)
__global__ void make_targets(uint32_t *t, uint64_t count, uint32_t n, int skew) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (uint64_t)gridDim.x * blockDim.x) {
        const double u = (double)(mix(k + 12345) >> 11) * 0x1p-53;
        t[k] = (uint32_t)(n * (skew ? u * u : u));
    }
}

// count the targets in [a, b) with global atomics (counts indexed by node)
__global__ void count_range(const uint32_t *__restrict__ t, uint64_t count, uint32_t a, uint32_t b, uint32_t *counts) {
    const uint4 *t4 = reinterpret_cast<const uint4 *>(t);
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count / 4; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(t4 + k);  // streaming (evict-first) read
        if (v.x - a < b - a) atomicAdd(counts + v.x, 1u);
        if (v.y - a < b - a) atomicAdd(counts + v.y, 1u);
        if (v.z - a < b - a) atomicAdd(counts + v.z, 1u);
        if (v.w - a < b - a) atomicAdd(counts + v.w, 1u);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t T = 1600000000ull;  // C4: 1.6e9 targets
    const uint32_t n = 100000000u;
    uint32_t *t, *c;
    CK(cudaMalloc(&t, T * 4));
    CK(cudaMalloc(&c, (size_t)n * 4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{");
    for (int skew = 0; skew < 2; ++skew) {
        make_targets<<<sms * 16, 256>>>(t, T, n, skew);
        CK(cudaDeviceSynchronize());
        for (int P : {1, 2, 3, 4, 6, 8}) {
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cudaMemset(c, 0, (size_t)n * 4));
                cudaEventRecord(e0);
                for (int k = 0; k < P; ++k) {
                    const uint32_t a = (uint32_t)((uint64_t)n * k / P), b = (uint32_t)((uint64_t)n * (k + 1) / P);
                    count_range<<<sms * 16, 512>>>(t, T, a, b, c);
                }
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("%s\"skew%d_P%d_ms\": %.3f", (skew || P > 1) ? ", " : "", skew, P, best);
        }
    }
    printf("}\n");
    return 0;
}
