#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k16cs(ulonglong2 *o, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        __stcs(o + i, make_ulonglong2(i, i ^ 0x5555ull));
}
__global__ void k16(ulonglong2 *o, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        o[i] = make_ulonglong2(i, i ^ 0x5555ull);
}
__global__ void k32(uint64_t *o, uint64_t n32) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n32; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t *p = o + 4 * i;
        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" :: "l"(p), "l"(i), "l"(i ^ 1), "l"(i ^ 2), "l"(i ^ 3) : "memory");
    }
}
__global__ void k32cs(uint64_t *o, uint64_t n32) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n32; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t *p = o + 4 * i;
        asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" :: "l"(p), "l"(i), "l"(i ^ 1), "l"(i ^ 2), "l"(i ^ 3) : "memory");
    }
}
int main() {
    const uint64_t bytes = 16ull << 30;
    void *b; cudaMalloc(&b, bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 148;
    for (int g : {4, 8, 16}) for (int which = 0; which < 4; ++which) {
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0);
            if (which == 0) k16cs<<<sms * g, 512>>>((ulonglong2 *)b, bytes / 16);
            if (which == 1) k16<<<sms * g, 512>>>((ulonglong2 *)b, bytes / 16);
            if (which == 2) k32<<<sms * g, 512>>>((uint64_t *)b, bytes / 32);
            if (which == 3) k32cs<<<sms * g, 512>>>((uint64_t *)b, bytes / 32);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
        }
        const char *nm[] = {"16B.cs", "16B", "32B", "32B.cs"};
        printf("grid %dx148 %s: %.1f GB/s\n", g, nm[which], bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
