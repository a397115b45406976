// parba_nodes.cuh -- node-granular kernels: the degree-sequence index (f4)
// and the option flags no_self_loops / no_parallel_edges (f3).
//
// Degree sequences (degreeseq.py): W[k] = m0 + sum of the degrees of nodes
// n0..n0+k-1 (exclusive scan on the device), W[n-n0] = m.  The owner of a
// position is found by rank over a bit vector with a one at every first edge
// of a node of degree >= 1 (parba_device.cuh: rank1_dev / node_of); the
// reference's binary search and deferred sort-and-merge lookups run here too
// (identical results, exercised by the parity tests).
//
// Option flags (generator.py:184-246): chains become node-granular.  With
// no_self_loops every edge of node v starts at r0 = 2*W_v (so all d chains of
// v coincide and resolve strictly before v); with no_parallel_edges edge i
// re-runs its chain under attempt-salted families 0, 1, 2, ... until its
// target is not among the node's earlier targets.  One thread walks one node
// in edge order -- exactly the reference's sequential rule -- while nodes
// run in parallel; a node's accepted targets live in the output it writes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "parba_device.cuh"

namespace parba {

// ---------------------------------------------------------------------------
// Degree-sequence index

// W[count] = W[count-1] + deg[count-1] (m0 when count == 0).
__global__ void degseq_last_kernel(const uint64_t *deg, uint64_t count, uint64_t m0, uint64_t *W) {
    if (blockIdx.x == 0 && threadIdx.x == 0) W[count] = count ? W[count - 1] + deg[count - 1] : m0;
}

// One bit per first edge of a node with degree >= 1 (degreeseq.py:118-124).
__global__ void rank_mark_kernel(const uint64_t *__restrict__ W, uint64_t count, ulonglong2 *rank) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = W[k], b = W[k + 1];
        if (b > a) atomicOr(reinterpret_cast<unsigned long long *>(&rank[a >> 6].x), 1ull << (a & 63));
    }
}

__global__ void rank_popc_kernel(const ulonglong2 *__restrict__ rank, uint64_t words, uint64_t *cnt) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x)
        cnt[w] = (uint64_t)__popcll(rank[w].x);
}

__global__ void rank_before_kernel(ulonglong2 *rank, const uint64_t *__restrict__ before, uint64_t words) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x)
        rank[w].y = before[w];
}

// owners[rank - 1] = node, for nodes of degree >= 1 (degreeseq.py:136-139).
__global__ void owners_kernel(const uint64_t *__restrict__ W, uint64_t count, uint64_t n0,
                              const ulonglong2 *__restrict__ rank, uint64_t *owners) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = W[k], b = W[k + 1];
        if (b > a) owners[rank1_dev(rank, a) - 1] = n0 + k;
    }
}

// Dense owner map: dense[pos - m0] = owning node of every generated position
// (one warp per node fills its edge span; spans are contiguous and disjoint).
__global__ void dense_fill_kernel(const uint64_t *__restrict__ W, uint64_t count, uint64_t m0, uint64_t n0,
                                  uint32_t *dense) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = warp; k < count; k += nwarps) {
        const uint64_t a = W[k], b = W[k + 1];
        for (uint64_t e = a + lane; e < b; e += 32) dense[e - m0] = (uint32_t)(n0 + k);
    }
}

__global__ void rank1_kernel(const ulonglong2 *__restrict__ rank, const uint64_t *__restrict__ es,
                             uint64_t count, uint64_t *out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = rank1_dev(rank, es[k]);
}

// node_of_edge_many (degreeseq.py:181-185): rank path.
__global__ void node_of_rank_kernel(DevParams p, const uint64_t *__restrict__ es, uint64_t count,
                                    uint64_t *out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = node_of(es[k], p);
}

// Rightmost k in [lo, hi) with W[k] <= e (W sorted; zero-degree nodes share
// their successor's W and are skipped by the right bias), degreeseq.py:188-196.
__device__ __forceinline__ uint64_t upper_bound_m1(const uint64_t *W, uint64_t lo, uint64_t hi, uint64_t e) {
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (__ldg(W + mid) <= e) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

// Degree-sequence chunking by edges: out[2k] = the first node v in
// [vlo, vhi] with W[v - n0] >= e0 + k * ce (k <= nch; the last is vhi),
// out[2k + 1] = W[v - n0].
__global__ void deg_chunk_bounds_kernel(const uint64_t *__restrict__ W, uint64_t n0, uint64_t vlo, uint64_t vhi,
                                        uint64_t e0, uint64_t ce, uint64_t nch, uint64_t *out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nch;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v;
        if (k == 0) {
            v = vlo;
        } else if (k == nch) {
            v = vhi;
        } else {  // lower bound: first index with W >= e
            const uint64_t e = e0 + k * ce;
            uint64_t lo = vlo - n0, hi = vhi - n0;
            while (lo < hi) {
                const uint64_t mid = lo + (hi - lo) / 2;
                if (__ldg(W + mid) < e) lo = mid + 1;
                else hi = mid;
            }
            v = lo + n0;
        }
        out[2 * k] = v;
        out[2 * k + 1] = __ldg(W + (v - n0));
    }
}

__global__ void node_of_bisect_kernel(DevParams p, const uint64_t *__restrict__ es, uint64_t count,
                                      uint64_t n_nodes, uint64_t *out) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        out[k] = p.n0 + upper_bound_m1(p.W, 0, n_nodes, es[k]);
}

// Deferred path (degreeseq.py:204-216, _kernels.py:101-118): keys sorted on
// the device (CUB radix sort), then each thread merges a run of kMergeRun
// consecutive sorted keys against W -- one binary search for the run's first
// key, then a forward walk (bounded; a long gap falls back to a search) --
// and scatters the owners back to the keys' original slots.
constexpr int kMergeRun = 64;
__global__ void merge_owner_kernel(DevParams p, const uint64_t *__restrict__ skeys,
                                   const uint64_t *__restrict__ sidx, uint64_t count, uint64_t n_nodes,
                                   uint64_t *out) {
    const uint64_t runs = (count + kMergeRun - 1) / kMergeRun;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < runs;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = r * kMergeRun, b = a + kMergeRun < count ? a + kMergeRun : count;
        uint64_t k = upper_bound_m1(p.W, 0, n_nodes, skeys[a]);
        for (uint64_t j = a; j < b; ++j) {
            const uint64_t e = skeys[j];
            int steps = 0;
            while (k + 1 < n_nodes && __ldg(p.W + k + 1) <= e && steps < 16) {
                ++k;
                ++steps;
            }
            if (steps == 16) k = upper_bound_m1(p.W, k, n_nodes, e);
            out[sidx[j]] = p.n0 + k;
        }
    }
}

__global__ void iota_kernel(uint64_t *v, uint64_t count) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        v[k] = k;
}

// out[0] = node owning position pos (m0 <= pos < m), out[1] = its first edge,
// out[2] = its end (first edge + degree).
__global__ void owner_span_kernel(DevParams p, uint64_t pos, uint64_t *out) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t v = node_of(pos, p);
        out[0] = v;
        out[1] = p.W[v - p.n0];
        out[2] = p.W[v - p.n0 + 1];
    }
}

// ---------------------------------------------------------------------------
// Option flags

constexpr int kFamilies = 256;  // retry families cached in shared memory
constexpr int kMemo = 288;      // memoised (r0, attempt) targets per small node (no_self_loops)
constexpr uint64_t kBigDegree = 256;  // no_parallel_edges: larger nodes use a hash set

struct NodeArgs {
    uint32_t no_self_loops, no_parallel_edges;
    uint32_t pre0;          // no_parallel_edges without no_self_loops: out already holds attempt 0
    uint64_t max_attempts;  // 0: 64 * degree (generator.py:205)
    uint32_t base_seed0, base_seed1;  // attempt a >= 1: salt a on the unsalted seeds
    uint64_t base_mult;
    uint32_t simple;
};

// One hash family of the retry sequence (HashConfig.with_attempt,
// hashing.py:69-85): attempt 0 is the configured family itself.
struct Family {
    uint32_t k0, k01;
    uint64_t mult;
};

__device__ __forceinline__ Family family_of(uint64_t attempt, const DevParams &p, const NodeArgs &na) {
    if (attempt == 0) return Family{p.k0, p.k01, p.mult};
    const uint32_t s0 = na.base_seed0 + (uint32_t)attempt;
    const uint32_t s1 = na.base_seed1 + (uint32_t)attempt * 0x9E3779B9u;
    Family f;
    f.k0 = crc32c_u64_bitwise(s0, 0);
    f.k01 = f.k0 ^ crc32c_u64_bitwise(s1, 0);
    f.mult = na.base_mult + 2ull * attempt * 0x9E3779B97F4A7C15ull;
    return f;
}

// h(r) under family f; tab = seed-free CRC tables (crc(0, .)): byte tables
// (8 KB; PARBA_NODE_CHUNKS=1: 5 chunk tables, 42 KB, measured 2x slower for
// both flags -- fewer resident CTAs), remainder on the FP64 pipe (mod_fp,
// exact for r < 2^52; the node paths require m <= 2^51; 20% faster than the
// integer-corrected mod_int for both flags).
#ifndef PARBA_NODE_CHUNKS
#define PARBA_NODE_CHUNKS 0
#endif
#ifndef PARBA_NODE_MODFP
#define PARBA_NODE_MODFP 1
#endif
__device__ __forceinline__ uint64_t hash_family(uint32_t tab, uint64_t r, const Family &f, bool simple) {
    if (simple) return __umul64hi(r * f.mult, r);
#if PARBA_NODE_CHUNKS
    const uint32_t c0 = crc_chunks<5>(tab, r) ^ f.k0;
#else
    const uint32_t c0 = crc_bytes<8>(tab, r) ^ f.k0;
#endif
#if PARBA_NODE_MODFP
    return mod_fp<uint64_t>(c0, c0 ^ f.k01, __ull2double_rn(r));
#else
    return mod_int(c0, c0 ^ f.k01, r);
#endif
}

// resolve_chain (generator.py:139-154): body at least once.
__device__ __forceinline__ uint64_t chain_family(uint32_t tab, uint64_t r, const Family &f, bool simple,
                                                 uint64_t stop, uint64_t &probes) {
    do {
        r = hash_family(tab, r, f, simple);
        ++probes;
    } while (!(r < stop || (r & 1ull) == 0));
    return r;
}

// Open-addressing set of a node's accepted targets (key t + 1; 0 = empty),
// capacity a power of two >= 2 * degree, in global scratch (big nodes).
__device__ __forceinline__ bool set_insert_if_absent(uint64_t *tab, uint32_t lg_cap, uint64_t t) {
    const uint64_t key = t + 1, mask = (1ull << lg_cap) - 1;
    uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> (64 - lg_cap);
    for (;;) {
        const uint64_t cur = tab[h];
        if (cur == key) return false;
        if (cur == 0) {
            tab[h] = key;
            return true;
        }
        h = (h + 1) & mask;
    }
}

// no_parallel_edges for one node (_node_edges_with_probes, generator.py:
// 199-217): edge i takes the first attempt a whose target is not among the
// node's accepted targets.  Membership: `set` (hash set, big nodes) or a scan
// of the node's output rows (small nodes).  With no_self_loops all edges of
// v share r0, so attempt a has the same target for every edge: targets and
// cumulative probe counts are memoised, and edge i starts at the attempt after
// edge i-1's (earlier ones stay rejected: the accepted set only grows) while
// adding the probes the reference spends re-walking them.
// no_self_loops membership scans of up to kLocalScan attempts read the memo
// in local memory; longer ones read the node's contiguous output rows (a
// thread's local array is interleaved across the warp: one cache line per
// element).
constexpr uint64_t kLocalScan = 32;

template <bool DEG, bool MEMO_SCAN = false>
__device__ __forceinline__ bool node_npe(uint64_t v, uint64_t first, uint64_t dv, uint64_t lo, ulonglong2 *out,
                                         uint64_t *set, uint32_t lg_cap, uint64_t *memo_t, uint64_t *memo_c,
                                         uint32_t memo_cap, const Family *fams, uint32_t tab, bool simple,
                                         const DevParams &p, const NodeArgs &na, uint64_t &probes,
                                         unsigned long long *fail_edge) {
    const bool nsl = na.no_self_loops != 0;
    const uint64_t cap = na.max_attempts ? na.max_attempts : 64 * dv;
    uint32_t n_memo = 0;
    uint64_t a_start = 0;
    for (uint64_t i = first; i < first + dv; ++i) {
        const uint64_t r0 = nsl ? 2 * first : 2 * i + 1;
        const uint64_t a0 = (nsl && a_start <= n_memo) ? a_start : 0;
        uint64_t pr_acc = (nsl && a0 > 0) ? memo_c[a0 - 1] : 0;
        uint64_t t = 0, a = a0;
        bool fresh = false;
        for (; a < cap; ++a) {
            if (na.pre0 && a == 0) {
                t = out[i - lo].y;  // attempt 0 = the plain edge, already generated (and its probes counted)
            } else if (nsl && a < n_memo) {
                t = memo_t[a];
                pr_acc = memo_c[a];
            } else {
                const Family f = a < kFamilies ? fams[a] : family_of(a, p, na);
                uint64_t pr = 0;
                t = target_of<false, true, false, DEG>(chain_family(tab, r0, f, simple, p.stop, pr), p);
                pr_acc += pr;
                if (nsl && a == n_memo && n_memo < memo_cap) {
                    memo_t[n_memo] = t;
                    memo_c[n_memo] = pr_acc;
                    ++n_memo;
                }
            }
            if (set) {
                fresh = set_insert_if_absent(set, lg_cap, t);
            } else if (MEMO_SCAN && nsl && a <= n_memo && a <= kLocalScan) {
                // no_self_loops: every earlier attempt b < a was tried by this
                // or an earlier edge and is accepted or a repeat of an accepted
                // target, so t is fresh iff it is the first occurrence in the
                // memoised attempt sequence (local memory, not the written rows)
                fresh = true;
                for (uint64_t b = 0; b < a; ++b)
                    if (memo_t[b] == t) {
                        fresh = false;
                        break;
                    }
            } else {
                fresh = true;
                for (uint64_t j = first; j < i; ++j)  // the node's accepted targets so far
                    if (out[j - lo].y == t) {
                        fresh = false;
                        break;
                    }
            }
            if (fresh) break;
        }
        probes += pr_acc;
        if (!fresh) {
            atomicMin(fail_edge, (unsigned long long)i);
            return false;
        }
        out[i - lo] = make_ulonglong2(v, t);
        a_start = a + 1;
    }
    return true;
}

// Node-kernel prologue: seed-free CRC chunk tables and the retry families.
#if PARBA_NODE_CHUNKS
#define PARBA_NODE_TABLES                                                                  \
    __shared__ uint32_t tabs_p[5 * 2048];                                                  \
    __shared__ uint32_t tab_bits[64];                                                      \
    build_chunk_tables_linear(tabs_p, 5, tab_bits)
#else
#define PARBA_NODE_TABLES                                                                  \
    __shared__ uint32_t tabs_p[8 * 256];                                                   \
    build_byte_tables(tabs_p, 8, 0u)
#endif
// no_self_loops-only kernels: no retry families
#define PARBA_NODE_PROLOGUE_NSL                                                            \
    PARBA_NODE_TABLES;                                                                     \
    __syncthreads();                                                                       \
    const uint32_t tab = opaque(smem_addr(tabs_p));                                        \
    const bool simple = na.simple != 0;                                                    \
    uint64_t probes = 0
#define PARBA_NODE_PROLOGUE                                                                \
    PARBA_NODE_TABLES;                                                                     \
    __shared__ Family fams[kFamilies];                                                     \
    if (na.no_parallel_edges)                                                              \
        for (int a_ = threadIdx.x; a_ < kFamilies; a_ += blockDim.x) fams[a_] = family_of(a_, p, na); \
    __syncthreads();                                                                       \
    const uint32_t tab = opaque(smem_addr(tabs_p));                                        \
    const bool simple = na.simple != 0;                                                    \
    uint64_t probes = 0

__device__ __forceinline__ void node_probes_flush(uint64_t probes, unsigned long long *probes_out) {
    if (probes_out) {
        for (int o = 16; o > 0; o >>= 1) probes += __shfl_xor_sync(0xffffffffu, probes, o);
        if ((threadIdx.x & 31) == 0 && probes) atomicAdd(probes_out, (unsigned long long)probes);
    }
}

template <bool DEG>
__device__ __forceinline__ void node_span(uint64_t v, const DevParams &p, uint64_t &first, uint64_t &dv) {
    if constexpr (DEG) {
        first = __ldg(p.W + (v - p.n0));
        dv = __ldg(p.W + (v - p.n0) + 1) - first;
    } else {
        first = p.m0 + (v - p.n0) * p.d;
        dv = p.d;
    }
}

// Edges of nodes [vlo, vhi) into out (row i - lo), honouring the flags
// (_node_edges_with_probes, generator.py:184-217), one thread per node.
// Under no_parallel_edges nodes of degree > big_deg are skipped here (they
// run in node_big_kernel with a hash set).  fail_edge receives the smallest
// edge index that found no fresh target (InfeasibleTargetsError).
template <bool DEG, bool MEMO_SCAN = false>  // MEMO_SCAN: both flags (see node_npe)
__global__ void __launch_bounds__(256)
node_kernel(DevParams p, NodeArgs na, uint64_t vlo, uint64_t vhi, uint64_t lo, uint64_t n_out, ulonglong2 *out,
            unsigned long long *probes_out, unsigned long long *fail_edge, uint64_t big_deg, const uint8_t *need) {
    PARBA_NODE_PROLOGUE;
    uint64_t memo_t[kMemo], memo_c[kMemo];
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t first, dv;
        node_span<DEG>(v, p, first, dv);
        if (dv == 0) continue;
        PARBA_CHECK(first - lo + dv <= n_out);
        if (!na.no_parallel_edges) {
            // no_self_loops alone: every edge of v runs the same chain
            uint64_t pr = 0;
            const Family f0{p.k0, p.k01, p.mult};
            const uint64_t r = chain_family(tab, 2 * first, f0, simple, p.stop, pr);
            probes += pr * dv;
            const uint64_t t = target_of<false, true, false, DEG>(r, p);
            for (uint64_t i = first; i < first + dv; ++i) out[i - lo] = make_ulonglong2(v, t);
            continue;
        }
        if (dv > big_deg || (need && !need[v - vlo])) continue;
        if (!MEMO_SCAN && na.pre0 && !need && dv <= 16) {  // (not compiled into the both-flags kernel)
            // attempt-0 targets (the plain pass's rows) pairwise distinct:
            // the node is final (npe_dup_kernel's rule, checked inline)
            uint64_t t[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = (uint64_t)k < dv ? out[first - lo + k].y : ~(uint64_t)k;
            bool dup = false;
#pragma unroll
            for (int a = 1; a < 16; ++a)
#pragma unroll
                for (int b = 0; b < a; ++b) dup |= t[a] == t[b];
            if (!dup) continue;
        }
        node_npe<DEG, MEMO_SCAN>(v, first, dv, lo, out, nullptr, 0, memo_t, memo_c, kMemo, fams, tab, simple, p, na,
                      probes, fail_edge);
    }
    node_probes_flush(probes, probes_out);
}

// no_self_loops alone: one chain per node (lane), and the warp's 32 nodes'
// rows written by the whole warp -- consecutive lanes store consecutive
// 16-byte rows (512-byte coalesced stores) instead of each lane striding
// through its own node's rows.  Row -> node: uniform d (<= 2^20) by the
// magic division; degree sequences by a binary search over the lanes'
// exclusive degree prefix (zero-degree lanes share the next lane's prefix,
// so the search lands on the owning lane).
template <bool DEG>
__global__ void __launch_bounds__(256)
node_nsl_kernel(DevParams p, NodeArgs na, uint64_t vlo, uint64_t vhi, uint64_t lo, ulonglong2 *out,
                unsigned long long *probes_out) {
    PARBA_NODE_PROLOGUE_NSL;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t vb = vlo + warp * 32; vb < vhi; vb += nwarps * 32) {  // warp-uniform trip count
        const uint64_t v = vb + lane;
        const uint32_t nact = vhi - vb < 32 ? (uint32_t)(vhi - vb) : 32u;
        uint64_t first = 0, dv = 0, t = 0;
        if (v < vhi) node_span<DEG>(v, p, first, dv);
        if (DEG ? dv != 0 : v < vhi) {
            uint64_t pr = 0;
            const Family f0{p.k0, p.k01, p.mult};
            const uint64_t r = chain_family(tab, 2 * first, f0, simple, p.stop, pr);
            probes += pr * dv;
            t = target_of<false, true, false, DEG>(r, p);
        }
        uint64_t first_b;  // first edge of the warp's first node
        uint64_t nrows;
        uint64_t excl = 0;  // DEG: rows of the lanes before this one
        if constexpr (DEG) {
            uint64_t inc = dv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= (uint32_t)o) inc += y;
            }
            excl = inc - dv;
            nrows = __shfl_sync(0xffffffffu, inc, 31);
            first_b = __shfl_sync(0xffffffffu, first, 0);
            if (v >= vhi) excl = nrows;  // inactive lanes sit past the end
        } else {
            nrows = (uint64_t)nact * p.d;
            first_b = p.m0 + (vb - p.n0) * p.d;
        }
        ulonglong2 *o = out + (first_b - lo);
        if constexpr (DEG) {
            for (uint64_t b = 0; b < nrows; b += 32) {
                const uint64_t rr = b + lane;
                const uint64_t rq = rr < nrows ? rr : nrows - 1;
                uint32_t k = 0;
#pragma unroll
                for (uint32_t st = 16; st > 0; st >>= 1) {
                    const uint64_t e = __shfl_sync(0xffffffffu, excl, k + st);
                    if (e <= rq) k += st;
                }
                const uint64_t tv = __shfl_sync(0xffffffffu, t, k);
                if (rr < nrows) __stcs(o + rr, make_ulonglong2(vb + k, tv));
            }
        } else {
            const uint32_t nr = (uint32_t)nrows;  // <= 32 * 2^20
            for (uint32_t b = 0; b < nr; b += 32) {
                const uint32_t rr = b + lane;
                const uint32_t k = magic_div32(rr < nr ? rr : nr - 1, p.div32);  // node of row rr
                const uint64_t tv = __shfl_sync(0xffffffffu, t, k);
                if (rr < nr) __stcs(o + rr, make_ulonglong2(vb + k, tv));
            }
        }
    }
    node_probes_flush(probes, probes_out);
}

// Degree counts under no_self_loops alone, fused: node v's dv edges all run
// the chain from 2*first, so they add dv to v and dv to their common target
// (both endpoints < K) -- two atomics per node, no edge rows in memory.
template <bool DEG, typename CountT>
__global__ void __launch_bounds__(256)
node_count_kernel(DevParams p, NodeArgs na, uint64_t vlo, uint64_t vhi, uint64_t K, CountT *counts,
                  unsigned long long *probes_out) {
    PARBA_NODE_PROLOGUE_NSL;
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t first, dv;
        node_span<DEG>(v, p, first, dv);
        if (dv == 0) continue;
        uint64_t pr = 0;
        const Family f0{p.k0, p.k01, p.mult};
        const uint64_t r = chain_family(tab, 2 * first, f0, simple, p.stop, pr);
        probes += pr * dv;
        const uint64_t t = target_of<false, true, false, DEG>(r, p);
        if (v < K) atomicAdd(counts + v, (CountT)dv);
        if (t < K) atomicAdd(counts + t, (CountT)dv);
    }
    node_probes_flush(probes, probes_out);
}

// Source endpoints of nodes [vlo, vhi) (all their edges): counts[v] += dv.
template <bool DEG, typename CountT>
__global__ void node_sources_kernel(DevParams p, uint64_t vlo, uint64_t vhi, CountT *counts) {
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t first, dv;
        node_span<DEG>(v, p, first, dv);
        if (dv) counts[v] += (CountT)dv;
    }
}

// no_parallel_edges for high-degree nodes: one thread per node with an
// open-addressing set of its targets (and its no_self_loops memo) in global
// scratch -- O(degree) per node instead of the scan's O(degree^2).  Node k of
// the launch is nodes[k] (or vlo + k); its scratch starts at off[k] (or k *
// per_node) words: set (2^lg words) then memo targets and cumulative probes.
template <bool DEG>
__global__ void __launch_bounds__(128)
node_big_kernel(DevParams p, NodeArgs na, const uint64_t *nodes, uint64_t vlo, uint64_t count,
                const uint64_t *off, uint64_t off_base, uint64_t per_node, uint64_t *scratch, uint64_t lo, uint64_t n_out,
                ulonglong2 *out, unsigned long long *probes_out, unsigned long long *fail_edge) {
    PARBA_NODE_PROLOGUE;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = nodes ? nodes[k] : vlo + k;
        uint64_t first, dv;
        node_span<DEG>(v, p, first, dv);
        PARBA_CHECK(first - lo + dv <= n_out);
        uint32_t lg = 1;
        while ((1ull << lg) < 2 * dv) ++lg;
        uint64_t *set = scratch + (off ? off[k] - off_base : k * per_node);
        for (uint64_t q = 0; q < (1ull << lg); ++q) set[q] = 0;
        const uint32_t memo_cap = (uint32_t)(2 * dv + 64);
        uint64_t *memo_t = set + (1ull << lg);
        node_npe<DEG>(v, first, dv, lo, out, set, lg, memo_t, memo_t + memo_cap, memo_cap, fams, tab, simple, p,
                      na, probes, fail_edge);
    }
    node_probes_flush(probes, probes_out);
}

// no_parallel_edges without no_self_loops, after the plain pass: a node
// whose attempt-0 targets are pairwise distinct is final (the sequential
// rule accepts every attempt 0).  need[v - vlo] = 1 marks the nodes the node
// kernels must re-run: a repeated target among <= 16 edges, or more edges.
template <bool DEG>
__global__ void npe_dup_kernel(DevParams p, uint64_t vlo, uint64_t vhi, uint64_t lo, const ulonglong2 *out,
                               uint8_t *need) {
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t first, dv;
        node_span<DEG>(v, p, first, dv);
        uint8_t f = dv > 16 ? 1 : 0;
        if (!f && dv >= 2) {
            uint64_t t[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = (uint64_t)k < dv ? out[first - lo + k].y : ~(uint64_t)k;
#pragma unroll
            for (int a = 1; a < 16; ++a)
#pragma unroll
                for (int b = 0; b < a; ++b) f |= t[a] == t[b] ? 1 : 0;
        }
        need[v - vlo] = f;
    }
}

// Scratch words of a big node: its set (power of two >= 2 * degree) + memo.
__host__ __device__ inline uint64_t node_big_words(uint64_t dv) {
    uint64_t c = 2;
    while (c < 2 * dv) c <<= 1;
    return c + 2 * (2 * dv + 64);
}

// Degree-sequence nodes of [vlo, vhi) with degree > big_deg: flags, then a
// CUB select; their scratch sizes for an exclusive scan.
__global__ void big_flags_kernel(DevParams p, uint64_t vlo, uint64_t vhi, uint64_t big_deg, uint8_t *flags) {
    for (uint64_t v = vlo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t dv = __ldg(p.W + (v - p.n0) + 1) - __ldg(p.W + (v - p.n0));
        flags[v - vlo] = dv > big_deg ? 1 : 0;
    }
}
__global__ void big_words_kernel(DevParams p, const uint64_t *nodes, uint64_t count, uint64_t *words) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = nodes[k];
        words[k] = node_big_words(__ldg(p.W + (v - p.n0) + 1) - __ldg(p.W + (v - p.n0)));
    }
}
__global__ void iota_from_kernel(uint64_t *v, uint64_t count, uint64_t start) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x)
        v[k] = start + k;
}

// count_block over stored pairs (analytics.py:44-48): both endpoints < K.
template <typename CountT>
__global__ void count_pairs_kernel(const ulonglong2 *__restrict__ pairs, uint64_t count, uint64_t K,
                                   CountT *counts) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const ulonglong2 e = pairs[k];
        if (e.x < K) atomicAdd(counts + e.x, (CountT)1);
        if (e.y < K) atomicAdd(counts + e.y, (CountT)1);
    }
}

}  // namespace parba
