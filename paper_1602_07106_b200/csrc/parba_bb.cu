// parba_bb.cu -- the Batagelj-Brandes edge array built as an ARRAY, not by
// chain recomputation: the device counterpart of the reference's sequential
// oracle bb_generate (oracle.py:45-107), which fills E left to right with
// E[2i] = source(i) and E[2i+1] = E[x], x = h(2i+1) in [0, 2i].
//
// The sequential fill reads E[x] written earlier; on the GPU every odd cell
// instead gets a pointer link[i] = h(2i+1) (one hash per edge) and the
// pointers are resolved by pointer jumping: while link[i] is an odd position
// 2j+1 >= 2m0, replace it by link[j] (whose cell E[2j+1] the sequential fill
// copied from).  Each pass at least halves every unresolved path, so a few
// passes (chains are geometric, mean 2) leave every link on an
// even (source) cell or in the seed region; then E[2i+1] = E[link[i]].
// This never runs a hash chain, so it checks the tile kernels' chain
// recomputation the way the reference's verify command checks its parallel
// path against the sequential fill (cli.py:332-351).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/parba_b200.h"
#include "parba_common.h"

using namespace parba;
using namespace parba::host;

namespace {

// E[j] = seed for j < 2m0; E[2i] = source(i); link[i - m0] = h(2i+1)
template <class Hash, bool DEG>
__global__ void __launch_bounds__(256) bb_link_kernel(DevParams p, uint64_t *__restrict__ E,
                                                      uint64_t *__restrict__ link) {
    __shared__ uint32_t tabs_p[Hash::kTableWords > 0 ? Hash::kTableWords : 1];
    Hash::build(tabs_p, p.k0);
    __syncthreads();
    const uint32_t tabs = opaque(smem_addr(tabs_p));
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (uint64_t j = t0; j < 2 * p.m0; j += stride) E[j] = __ldg(p.seed + j);
    for (uint64_t i = p.m0 + t0; i < p.m; i += stride) {
        E[2 * i] = source_of<false, true, DEG>(i, p);
        link[i - p.m0] = Hash::probe(tabs, 2 * i + 1, p);
    }
}

// One pointer-jumping pass (in place: any link value read is a valid
// shortcut of the same path, whichever pass wrote it).
__global__ void __launch_bounds__(256) bb_jump_kernel(uint64_t m0, uint64_t n_links, uint64_t *link,
                                                      unsigned int *changed) {
    bool any = false;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_links;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = link[k];
        if ((x & 1) && x >= 2 * m0) {
            x = link[(x >> 1) - m0];  // E[2j+1] = E[link[j]], j = (x - 1) / 2
            link[k] = x;
            any = true;
        }
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(changed, 1u);
}

__global__ void __launch_bounds__(256) bb_gather_kernel(uint64_t m0, uint64_t m, uint64_t *E,
                                                        const uint64_t *__restrict__ link) {
    for (uint64_t i = m0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        E[2 * i + 1] = E[link[i - m0]];  // an even (source) cell or a seed cell
}

template <class Hash>
int bb_link(const parba_params_t *p, const DevParams &dp, uint64_t *E, uint64_t *link, cudaStream_t st) {
    const unsigned g = grid_for(p->m - p->m0 > 2 * p->m0 ? p->m - p->m0 : 2 * p->m0, 256);
    if (is_deg(p)) bb_link_kernel<Hash, true><<<g, 256, 0, st>>>(dp, E, link);
    else bb_link_kernel<Hash, false><<<g, 256, 0, st>>>(dp, E, link);
    CUDA_TRY(cudaGetLastError());
    return PARBA_OK;
}

}  // namespace

extern "C" {

int parba_bb_fill(const parba_params_t *p, uint64_t *E, uint64_t *link, unsigned int *flag, int *passes,
                  void *stream) {
    int rc = validate(p);
    if (rc) return rc;
    if (p->flags) return fail(PARBA_EINVAL, "the sequential oracle supports plain mode only");
    if (!E || !flag || (p->m > p->m0 && !link)) return fail(PARBA_EINVAL, "NULL buffer");
    cudaStream_t st = (cudaStream_t)stream;
    const DevParams dp = make_dev(p);
    if (p->hash_kind == PARBA_HASH_SIMPLE) rc = bb_link<HashSimple<false>>(p, dp, E, link, st);
    else rc = bb_link<HashCrcBytes>(p, dp, E, link, st);
    if (rc) return rc;
    const uint64_t nl = p->m - p->m0;
    int k = 0;
    for (; nl > 0; ++k) {  // until a pass changes nothing
        CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(unsigned int), st));
        bb_jump_kernel<<<grid_for(nl, 256), 256, 0, st>>>(p->m0, nl, link, flag);
        CUDA_TRY(cudaGetLastError());
        unsigned int h = 0;
        CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (!h) break;
        if (k > 64) return fail(PARBA_ECUDA, "pointer jumping did not converge");
    }
    if (passes) *passes = k + (nl > 0);
    if (nl) {
        bb_gather_kernel<<<grid_for(nl, 256), 256, 0, st>>>(p->m0, p->m, E, link);
        CUDA_TRY(cudaGetLastError());
    }
    return PARBA_OK;
}

}  // extern "C"
