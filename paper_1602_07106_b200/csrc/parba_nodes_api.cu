// parba_nodes_api.cu -- the node-granular half of the C ABI: the degree-
// sequence index entry points (f4: prefix, rank directory, dense owner map,
// owner lookups) and the host side of the option-flag paths (f3: node
// boundaries, the node kernels, infeasible-target reporting, flag counts).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "../../include/parba_b200.h"
#include "parba_common.h"
#include "parba_nodes.cuh"

using namespace parba;
using namespace parba::host;

namespace parba {
namespace host {

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


// The node kernels hash chain values < 2m with 5 chunk tables and the FP64
// remainder (hash_family): every value must stay below 2^52.
constexpr uint64_t kNodeMaxEdges = 1ull << 51;

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
    thrust::counting_iterator<uint64_t> ids(vlo);
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

// PARBA_EINFEASIBLE with the reference's message when a node kernel
// recorded a failing edge (InfeasibleTargetsError, generator.py:209-213).
int report_infeasible(const parba_params_t *p, const DevParams &dp, const uint64_t *fail_edge, cudaStream_t st) {
    int rc;
    uint64_t edge;
    rc = read_u64s(fail_edge, &edge, 1, st);
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

// Edges of nodes [vlo, vhi) (first edge lo) into out, honouring the flags;
// synchronises st to report an infeasible node (InfeasibleTargetsError).
// fail_ext: a caller-owned failing-edge word (atomicMin, initialised to
// UINT64_MAX) that the caller reports once after several calls; otherwise
// the failure is reported here (one device sync).
#ifndef PARBA_INLINE_DUP
#define PARBA_INLINE_DUP 1
#endif
int generate_nodes(const parba_params_t *p, const DevParams &dp, uint64_t vlo, uint64_t vhi, uint64_t lo,
                   uint64_t hi, uint64_t *out, unsigned long long *probes, cudaStream_t st,
                   unsigned long long *fail_ext) {
    if (vhi <= vlo) return PARBA_OK;
    if (p->m > kNodeMaxEdges) return fail(PARBA_EINVAL, "option flags support m <= 2^51 edges (m = %llu)",
                                          (unsigned long long)p->m);
    NodeArgs na{};
    na.no_self_loops = (p->flags & PARBA_FLAG_NO_SELF_LOOPS) ? 1u : 0u;
    na.no_parallel_edges = (p->flags & PARBA_FLAG_NO_PARALLEL_EDGES) ? 1u : 0u;
    na.max_attempts = p->max_attempts;
    na.base_seed0 = p->base_seed0;
    na.base_seed1 = p->base_seed1;
    na.base_mult = p->base_mult;
    na.simple = p->hash_kind == PARBA_HASH_SIMPLE ? 1u : 0u;
    // no_parallel_edges alone: attempt 0 of every edge is the plain edge, so
    // the tile kernel generates them all first (full speed, probes counted)
    // and the node kernels only re-run the edges whose target repeats
    na.pre0 = (na.no_parallel_edges && !na.no_self_loops) ? 1u : 0u;
    if (na.pre0) {
        int rc0 = launch_store(p, dp, lo, hi, out, probes, st);
        if (rc0) return rc0;
    }
    AsyncBuf fe, need;
    int rc = PARBA_OK;
    if (!fail_ext) {
        if ((rc = fe.alloc(sizeof(unsigned long long), st))) return rc;
        CUDA_TRY(cudaMemsetAsync(fe.p, 0xFF, sizeof(unsigned long long), st));
    }
    const unsigned grid = grid_for(vhi - vlo, 256);
    // PARBA_INLINE_DUP: the node kernel checks the attempt-0 rows of nodes of
    // degree <= 16 itself (one pass over the rows instead of npe_dup_kernel +
    // the node kernel); larger nodes always re-run
    if (na.pre0 && !PARBA_INLINE_DUP) {  // nodes whose attempt-0 targets are already distinct are final
        if ((rc = need.alloc(vhi - vlo, st))) return rc;
        if (is_deg(p))
            npe_dup_kernel<true><<<grid, 256, 0, st>>>(dp, vlo, vhi, lo, (const ulonglong2 *)out, (uint8_t *)need.p);
        else
            npe_dup_kernel<false><<<grid, 256, 0, st>>>(dp, vlo, vhi, lo, (const ulonglong2 *)out, (uint8_t *)need.p);
        CUDA_TRY(cudaGetLastError());
    }
    const uint64_t big = na.no_parallel_edges ? kBigDegree : UINT64_MAX;
    unsigned long long *fep = fail_ext ? fail_ext : (unsigned long long *)fe.p;
    const uint8_t *needp = (const uint8_t *)need.p;
    if (na.no_self_loops && !na.no_parallel_edges && (is_deg(p) || p->d <= (1u << 20))) {
        if (is_deg(p))
            node_nsl_kernel<true><<<grid, 256, 0, st>>>(dp, na, vlo, vhi, lo, (ulonglong2 *)out, probes);
        else
            node_nsl_kernel<false><<<grid, 256, 0, st>>>(dp, na, vlo, vhi, lo, (ulonglong2 *)out, probes);
        CUDA_TRY(cudaGetLastError());
        return fail_ext ? PARBA_OK : report_infeasible(p, dp, (const uint64_t *)fe.p, st);
    }
    const bool both = na.no_self_loops && na.no_parallel_edges;
    auto args = [&](auto kern) {
        kern<<<grid, 256, 0, st>>>(dp, na, vlo, vhi, lo, hi - lo, (ulonglong2 *)out, probes, fep, big, needp);
    };
    if (is_deg(p)) both ? args(node_kernel<true, true>) : args(node_kernel<true, false>);
    else both ? args(node_kernel<false, true>) : args(node_kernel<false, false>);
    CUDA_TRY(cudaGetLastError());
    if (na.no_parallel_edges) {
        rc = generate_big_nodes(p, dp, na, vlo, vhi, lo, hi, out, probes, fep, st);
        if (rc) return rc;
    }
    return fail_ext ? PARBA_OK : report_infeasible(p, dp, (const uint64_t *)fe.p, st);
}

// Degree counts of [lo, hi) with option flags: node-aligned chunks generated
// into scratch, then counted (both endpoints < K).
#ifndef PARBA_COUNT_CHUNK_LG
#define PARBA_COUNT_CHUNK_LG 26
#endif
template <typename CountT>
int count_nodes(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                CountT *counts, unsigned long long *probes, cudaStream_t st) {
    if (p->m > kNodeMaxEdges) return fail(PARBA_EINVAL, "option flags support m <= 2^51 edges (m = %llu)",
                                          (unsigned long long)p->m);
    uint64_t vlo, vhi;
    int rc = boundary_node(p, dp, lo, &vlo, st);
    if (!rc) rc = boundary_node(p, dp, hi, &vhi, st);
    if (rc) return rc;
    if (vhi <= vlo) return PARBA_OK;
    if (!(p->flags & PARBA_FLAG_NO_PARALLEL_EDGES)) {  // no_self_loops alone: fused, per node
        NodeArgs na{};
        na.no_self_loops = 1u;
        na.simple = p->hash_kind == PARBA_HASH_SIMPLE ? 1u : 0u;
        const unsigned grid = grid_for(vhi - vlo, 256);
        if (is_deg(p))
            node_count_kernel<true, CountT><<<grid, 256, 0, st>>>(dp, na, vlo, vhi, K, counts, probes);
        else
            node_count_kernel<false, CountT><<<grid, 256, 0, st>>>(dp, na, vlo, vhi, K, counts, probes);
        CUDA_TRY(cudaGetLastError());
        return PARBA_OK;
    }
    // node-aligned chunks of about 2^PARBA_COUNT_CHUNK_LG edges (16 B each in
    // scratch); the chunk bounds cost at most one device sync and a failing
    // edge is reported once at the end, so the chunks queue back to back.
    // Chunk c: nodes [bv[c], bv[c + 1]), edges [be[c], be[c + 1]).
    uint64_t ce = 1ull << PARBA_COUNT_CHUNK_LG;
    if (const char *e = getenv("PARBA_COUNT_CHUNK_EDGES")) {  // tests: many small chunks
        const unsigned long long x = strtoull(e, nullptr, 10);
        if (x > 0) ce = x;
    }
    std::vector<uint64_t> bv, be;
    if (is_deg(p)) {  // cut by edges: lower bounds of lo + k * ce in W, one sync
        const uint64_t nch = (hi - lo + ce - 1) / ce;
        AsyncBuf bnd;
        if ((rc = bnd.alloc((nch + 1) * 16, st))) return rc;
        deg_chunk_bounds_kernel<<<grid_for(nch + 1, 256), 256, 0, st>>>(p->degree_prefix, p->n0, vlo, vhi, lo, ce,
                                                                        nch, (uint64_t *)bnd.p);
        CUDA_TRY(cudaGetLastError());
        std::vector<uint64_t> h(2 * (nch + 1));
        if ((rc = read_u64s((const uint64_t *)bnd.p, h.data(), h.size(), st))) return rc;
        for (uint64_t k = 0; k <= nch; ++k)
            if (bv.empty() || h[2 * k] > bv.back()) {
                bv.push_back(h[2 * k]);
                be.push_back(h[2 * k + 1]);
            }
    } else {
        const uint64_t step = ce / p->d > 0 ? ce / p->d : 1;
        for (uint64_t v = vlo;; v = v + step < vhi ? v + step : vhi) {
            bv.push_back(v);
            be.push_back(node_first_edge(p, v));
            if (v == vhi) break;
        }
    }
    AsyncBuf fe;
    if ((rc = fe.alloc(sizeof(unsigned long long), st))) return rc;
    CUDA_TRY(cudaMemsetAsync(fe.p, 0xFF, sizeof(unsigned long long), st));
    unsigned long long *fep = (unsigned long long *)fe.p;
    for (size_t c = 0; c + 1 < bv.size(); ++c) {
        const uint64_t v = bv[c], v1 = bv[c + 1];
        const uint64_t a = be[c], b = be[c + 1];
        if (b <= a) continue;
        AsyncBuf scratch;
        if ((rc = scratch.alloc((b - a) * 16, st))) return rc;
        if ((rc = generate_nodes(p, dp, v, v1, a, b, (uint64_t *)scratch.p, probes, st, fep))) return rc;
        if (K == 0) continue;
        // large K: targets through the partitioned count, sources per node
        bool done = false;
        if ((rc = count_rows_partitioned((const ulonglong2 *)scratch.p, b - a, K, counts, &done, st))) return rc;
        if (done) {
            const uint64_t s1 = v1 < K ? v1 : K;
            if (v < s1) {
                if (is_deg(p))
                    node_sources_kernel<true, CountT><<<grid_for(s1 - v, 256), 256, 0, st>>>(dp, v, s1, counts);
                else
                    node_sources_kernel<false, CountT><<<grid_for(s1 - v, 256), 256, 0, st>>>(dp, v, s1, counts);
                CUDA_TRY(cudaGetLastError());
            }
        } else {
            count_pairs_kernel<CountT><<<grid_for(b - a, 256), 256, 0, st>>>((const ulonglong2 *)scratch.p, b - a,
                                                                             K, counts);
            CUDA_TRY(cudaGetLastError());
        }
    }
    return report_infeasible(p, dp, (const uint64_t *)fe.p, st);
}

int count_nodes_u64(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                    unsigned long long *counts, unsigned long long *probes, cudaStream_t st) {
    return count_nodes<unsigned long long>(p, dp, lo, hi, K, counts, probes, st);
}
int count_nodes_u32(const parba_params_t *p, const DevParams &dp, uint64_t lo, uint64_t hi, uint64_t K,
                    uint32_t *counts, unsigned long long *probes, cudaStream_t st) {
    return count_nodes<uint32_t>(p, dp, lo, hi, K, counts, probes, st);
}

}  // namespace host
}  // namespace parba

extern "C" {

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

}  // extern "C"
