/*
 * parba_b200.h -- C ABI of the B200-native Barabasi-Albert edge generator
 * (Sanders & Schulz, arXiv 1602.07106).
 *
 * Every entry point replaces one seam of the reference package `parba`
 * (/root/reference/pkg/src/parba/...; file:line cited per function).  The
 * signatures carry plain pointers and sizes only: no torch, no C++ types.
 *
 * Conventions
 *   - Return value: PARBA_OK (0) or a PARBA_E* code; parba_last_error()
 *     returns a thread-local, human-readable description of the last failure.
 *     Bad parameters map to ParameterError in the Python layer
 *     (errors.py:6-7), CUDA failures to GenerationError (errors.py:27-28).
 *   - Device entry points (no `_host` suffix): every pointer is a DEVICE
 *     pointer on the current CUDA device, owned by the caller; the launch is
 *     asynchronous on `stream` (a cudaStream_t, NULL = legacy default).
 *   - `probes`, when non-NULL, is a device u64 that is INCREMENTED by the
 *     total number of hash evaluations (RunStats.hash_probes, driver.py:50-55).
 *   - Count buffers ACCUMULATE (+=), so partial ranges merge the way
 *     Consumer.merge does (analytics.py:78-82).
 *   - `_host` entry points take HOST buffers, run on `device`, and return
 *     after the result is in host memory (blocking).
 *   - Thread-safe per (device, stream).
 */
#ifndef PARBA_B200_H
#define PARBA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARBA_OK 0
#define PARBA_EINVAL 1   /* parameter / range error  -> ParameterError   */
#define PARBA_ECUDA 2    /* CUDA runtime / launch error -> GenerationError */
#define PARBA_ENOMEM 3   /* device or pinned allocation failed            */

#define PARBA_EINFEASIBLE 4 /* no fresh target within max_attempts -> InfeasibleTargetsError (errors.py:19-24) */

#define PARBA_HASH_CRC 0u    /* HashKind.CRC    (hashing.py:43-45, 119-125) */
#define PARBA_HASH_SIMPLE 1u /* HashKind.SIMPLE (hashing.py:128-138)        */

/* GenParams option flags (generator.py:61-62, 184-246). */
#define PARBA_FLAG_NO_SELF_LOOPS 1u
#define PARBA_FLAG_NO_PARALLEL_EDGES 2u

/* Owner-lookup methods of a degree sequence (generator.py:30, 248-255). */
#define PARBA_RESOLVE_RANK 0u
#define PARBA_RESOLVE_BISECT 1u
#define PARBA_RESOLVE_DEFERRED 2u

/* Graph family = GenParams (generator.py:50-110): a uniform degree d or a
 * degree sequence, the seed graph, the option flags, plus the effective hash
 * constants of its HashConfig (hashing.py:48-85).  Zero-initialise the
 * fields after seed_edges for the plain uniform-d family. */
typedef struct parba_params {
    uint64_t n;            /* node count                                   */
    uint64_t d;            /* uniform out-degree (>= 1)                    */
    uint64_t n0;           /* seed nodes                                   */
    uint64_t m0;           /* seed edges (= len(seed_edges)/2)             */
    uint64_t m;            /* m0 + (n - n0) * d                            */
    uint32_t hash_kind;    /* PARBA_HASH_*                                 */
    uint32_t crc_seed0;    /* HashConfig.crc_seeds()[0] (salt folded in)   */
    uint32_t crc_seed1;    /* HashConfig.crc_seeds()[1]                    */
    uint32_t reserved;     /* must be 0                                    */
    uint64_t simple_mult;  /* HashConfig.simple_multiplier()               */
    const uint64_t *seed_edges; /* DEVICE pointer to 2*m0 node IDs (NULL iff m0 == 0) */
    /* option flags (f3) */
    uint32_t flags;        /* PARBA_FLAG_* (both require m0 >= 1)          */
    uint32_t reserved2;    /* must be 0                                    */
    uint64_t max_attempts; /* no_parallel_edges retry cap; 0 = 64 * degree */
    uint32_t base_seed0;   /* seed0 & 0xFFFFFFFF: retry attempt a >= 1 uses  */
    uint32_t base_seed1;   /* seed1 & 0xFFFFFFFF  the family with salt a     */
    uint64_t base_mult;    /* HashConfig.multiplier    (with_attempt, hashing.py:69-85) */
    /* degree sequence (f4): d == 0 and these three set (DEVICE pointers,
     * built by parba_degseq_prefix / parba_degseq_rank); m = W[n - n0]   */
    const uint64_t *degree_prefix; /* W: n - n0 + 1 entries               */
    const void *rank;              /* rank directory, (m + 63) / 64 x 16 B */
    const uint64_t *owners;        /* rank -> node; NULL iff every degree >= 1 */
    const uint32_t *dense_owner;   /* optional (NULL): owning node of every position
                                      m0..m-1 (parba_degseq_dense; n < 2^32), 4 B
                                      per edge: one load per owner lookup */
} parba_params_t;

/* Library / ABI version (major*10000 + minor*100 + patch). */
int parba_version(void);
/* Thread-local description of the last error ("" if none). */
const char *parba_last_error(void);
/* Number of visible CUDA devices (0 when none); never fails. */
int parba_device_count(void);

/* Elementwise position hash out[k] = h(r[k]) -- hash_many / hash_value
 * (hashing.py:141-145, 194-198).  Requires r[k] >= 1 (checked by caller). */
int parba_hash(const parba_params_t *p, const uint64_t *r, uint64_t count, uint64_t *out,
               void *stream);

/* crc32c_u64_many (hashing.py:105-116, 158-165): out[k] = raw reflected
 * CRC32-C of the 8 little-endian bytes of words[k] accumulated on seed (no
 * inversion), widened to u64. */
int parba_crc32c(uint32_t seed, const uint64_t *words, uint64_t count, uint64_t *out, void *stream);
/* mulhi_u64 (hashing.py:168-176): out[k] = high 64 bits of a[k] * b[k]. */
int parba_mulhi_u64(const uint64_t *a, const uint64_t *b, uint64_t count, uint64_t *out, void *stream);

/* resolve_chain_block (_kernels.py:121-135): out[k] = terminal r of the
 * chain started at r0[k] (body at least once; stop when r < stop_below or r
 * even).  r0 is not modified; out may not alias r0. */
int parba_resolve_chains(const parba_params_t *p, const uint64_t *r0, uint64_t count,
                         uint64_t stop_below, uint64_t *out, unsigned long long *probes,
                         void *stream);

/* generate_block, plain path (generator.py:258-270, 288-325): rows
 * (source, target) of edges lo..hi-1 into out_pairs[2*(hi-lo)] (u64,
 * 16-byte aligned) -- the same bytes as the reference's (hi-lo, 2) uint64
 * array and as its binary edge file (cli.py:121-139).  m0 <= lo <= hi <= m. */
int parba_generate(const parba_params_t *p, uint64_t lo, uint64_t hi, uint64_t *out_pairs,
                   unsigned long long *probes, void *stream);

/* Store mode, targets column only: targets[i - lo] = (uint32) target of
 * edge i for lo <= i < hi (the source is the closed form (i - m0) / d + n0,
 * generator.py:163-169).  4 B per edge instead of 16: the host-array path
 * (parba_generate_host) moves this over PCIe and fills the pairs on the
 * host.  CRC hash, uniform degree, no option flags, n <= 2^32. */
int parba_generate_targets(const parba_params_t *p, uint64_t lo, uint64_t hi, uint32_t *targets,
                           unsigned long long *probes, void *stream);

/* generate_edge on an arbitrary ID list (generator.py:172-181):
 * out_pairs[2k], out_pairs[2k+1] = edge ids[k].  Every id in [m0, m). */
int parba_edges_at(const parba_params_t *p, const uint64_t *ids, uint64_t count,
                   uint64_t *out_pairs, unsigned long long *probes, void *stream);

/* Fused generate_block + DegreeCountConsumer (analytics.py:44-48, 61-82):
 * counts[v] += degree contribution of edges lo..hi-1 to node v, for v < K
 * (both endpoints; a self-loop counts 2).  E is never stored. */
int parba_degree_window(const parba_params_t *p, uint64_t lo, uint64_t hi, uint64_t K,
                        unsigned long long *counts, unsigned long long *probes, void *stream);

/* Full-histogram variant (degree_counts with K = n, analytics.py:85-99):
 * counts[v] += contribution for every v < n, uint32 counters. */
int parba_degree_full(const parba_params_t *p, uint64_t lo, uint64_t hi, uint32_t *counts,
                      unsigned long long *probes, void *stream);

/* count_block on device (analytics.py:44-48): counts[ids[k]] += 1 for
 * ids[k] < K.  Folds seed edges into a count (count_seed_edges,
 * analytics.py:51-52). */
int parba_count_ids(const uint64_t *ids, uint64_t count, uint64_t K, unsigned long long *counts,
                    void *stream);

/* ---- Degree sequences (f4; degreeseq.py) ------------------------------
 * build_prefix (degreeseq.py:87-115): W[k] = m0 + degrees[0] + ... +
 * degrees[k-1] for k <= count (W[count] = m), by a device scan.  The caller
 * validates the degrees (non-negative, no overflow, m < 2^58). */
int parba_degseq_prefix(const uint64_t *degrees, uint64_t count, uint64_t m0, uint64_t *W, void *stream);
/* build_rank_bits (degreeseq.py:118-151): rank directory over positions
 * [0, m) -- ((m + 63) / 64) 16-byte entries {start bits, ones before} -- and,
 * when owners != NULL, owners[j] = node of the j-th node with degree >= 1.
 * n_ones (host, optional) receives the number of such nodes. */
int parba_degseq_rank(const uint64_t *W, uint64_t count, uint64_t m, uint64_t n0, void *rank,
                      uint64_t *owners, uint64_t *n_ones, void *stream);
/* Optional dense owner map for faster generation: dense[e - m0] = owner(e)
 * for every generated position (m - m0 entries of 4 bytes; needs n < 2^32).
 * Same results as the rank directory. */
int parba_degseq_dense(const uint64_t *W, uint64_t count, uint64_t m0, uint64_t n0, uint32_t *dense,
                       void *stream);
/* rank1_many (degreeseq.py:154-162): out[k] = ones at positions 0..es[k]. */
int parba_rank1(const void *rank, const uint64_t *es, uint64_t count, uint64_t *out, void *stream);
/* node_of_edge_many / node_of_edge_bisect_many / owners_of_edges_deferred
 * (degreeseq.py:165-216): out[k] = owning node of position es[k] (every
 * es[k] in [m0, m)), by PARBA_RESOLVE_* -- identical results. */
int parba_node_of_edges(const parba_params_t *p, const uint64_t *es, uint64_t count, uint64_t *out,
                        uint32_t method, void *stream);

/* ---- Option flags (f3) --------------------------------------------------
 * With p->flags set, parba_generate / parba_degree_window / parba_degree_full
 * are node-granular: lo and hi must be node boundaries (hi may be m), as in
 * generate_block (generator.py:272-302), and the call synchronises `stream`
 * to report PARBA_EINFEASIBLE (no fresh target within max_attempts).
 * generate_node_edges(v) = parba_generate over [W_v, W_v + d_v). */

/* count_block over stored pairs (analytics.py:44-48): counts[x] += 1 for
 * each endpoint x < K of pairs[0..count). */
int parba_count_pairs(const uint64_t *pairs, uint64_t count, uint64_t K, unsigned long long *counts,
                      void *stream);

/* Host-buffer entry points (blocking; uniform degree only -- a degree
 * sequence's index lives on the device).  generate_block into a host array
 * out_pairs[2*(hi-lo)]: the device generates in chunks while earlier chunks
 * stream back over PCIe (pinned host memory gets full DMA speed). */
int parba_generate_host(const parba_params_t *p_host_seed, uint64_t lo, uint64_t hi,
                        uint64_t *out_pairs_host, uint64_t *probes_host, int device);
/* Positional binary edge file (EdgeFileWriter / _pwrite_all, cli.py:109-145):
 * rows (source, target) of edges lo..hi-1 written into the open file `fd`
 * at byte offset 16*(i - base_edge) (base_edge = the file's first edge, the
 * reference's m0).  The file must already span the range (ftruncate).  The
 * range is mapped (MAP_SHARED) and filled by the host-array pipeline of
 * parba_generate_host, so rows go straight into the page cache from many
 * host threads instead of through one pwrite copy.  Blocking. */
int parba_write_binary(const parba_params_t *p_host_seed, uint64_t lo, uint64_t hi, int fd,
                       uint64_t base_edge, uint64_t *probes_host, int device);
/* degree_counts for [lo,hi) into host int64 counts[K] (+=). */
int parba_degree_window_host(const parba_params_t *p_host_seed, uint64_t lo, uint64_t hi,
                             uint64_t K, int64_t *counts_host, uint64_t *probes_host, int device);

/* Single-process multi-GPU run over [m0, m) (parba_multi_run;
 * the fork workers + Consumer.merge of driver.py:210-270, analytics.py:78-99):
 * equal contiguous shards on devs[0..ndev), one host thread per distinct
 * device (a device may repeat: its shards run back to back into one
 * histogram).
 *   PARBA_MULTI_STORE   out_host = host u64 pairs [2*(m - m0)] (edge i at row i - m0)
 *   PARBA_MULTI_WINDOW  out_host = host int64 counts[K], +=
 *   PARBA_MULTI_FULL    out_host = host int64 counts[n], += (needs 2m < 2^32)
 *   PARBA_MULTI_DISCARD out_host unused (probes and time only)
 * The distinct devices' histograms are summed by one ncclReduce (SUM, root
 * devs[0]; NCCL loaded at run time) -- the DegreeCountConsumer.merge of
 * analytics.py:78-82.  PARBA_MULTI_FULL on several devices with peer access
 * takes the owner-routed count instead (parba_degree_full_routed: device g
 * owns nodes [g * slice, (g + 1) * slice), the count kernels add into the
 * owners over NVLink, every device copies its own slice to the host), when
 * it applies to every shard; PARBA_MULTI_ROUTED=0 keeps the ncclReduce.  probes_host and device_seconds (max over devices of
 * generation + reduction) are optional.  Uniform degree only (host entry
 * point); option flags cut at node boundaries. */
#define PARBA_MULTI_STORE 0
#define PARBA_MULTI_WINDOW 1
#define PARBA_MULTI_FULL 2
#define PARBA_MULTI_DISCARD 3
int parba_multi_run(const parba_params_t *p_host_seed, int ndev, const int *devs, int mode, uint64_t K,
                    void *out_host, uint64_t *probes_host, double *device_seconds);
/* The same with explicit shards: shard s = edges [los[s], his[s]) on device
 * devs[s] (driver.run's worker batches, driver.py:161-207);
 * probes_per_shard[s] (optional) = that shard's hash probes
 * (WorkerStats.probes, driver.py:41-47).  Under option flags every cut must
 * be a node boundary. */
int parba_multi_run_shards(const parba_params_t *p_host_seed, int nshards, const int *devs,
                           const uint64_t *los, const uint64_t *his, int mode, uint64_t K, void *out_host,
                           uint64_t *probes_per_shard, double *device_seconds);

/* ---- Owner-routed full histogram: the histogram reduce fused into the count
 * (the N-GPU form of analytics.py:78-99: every worker counts its edge range,
 * DegreeCountConsumer.merge sums the arrays).  Node v's uint32 counter lives
 * on owner g = v / slice_nodes at slices[g][v - g * slice_nodes]; slices[g]
 * is a device pointer valid on the CURRENT device -- local memory, a peer
 * mapping (cudaDeviceEnablePeerAccess) or an IPC mapping (parba_ipc_open) of
 * owner g's memory over NVLink.  The count kernels add each bucket's
 * counters (closed-form sources included) straight into the owners' slices
 * with red.add as the bucket is counted, so the reduce-scatter of the
 * histograms overlaps the counting and no n-word array per GPU is summed
 * afterwards.  All workers call this with the same slice table; the owners
 * zero their slices before any worker starts and read them after every
 * worker's stream has drained (the caller's barriers).  slice_nodes: a
 * multiple of 65536 with nowners * slice_nodes >= n; nowners <= 16.
 * parba_degree_full_routed_ok = 1 when the path applies to [lo, hi) (plain
 * uniform-degree family, n >= 2^25, a shard of >= 2^22 edges): otherwise use
 * parba_degree_full and a reduce. */
int parba_degree_full_routed_ok(const parba_params_t *p, uint64_t lo, uint64_t hi);
int parba_degree_full_routed(const parba_params_t *p, uint64_t lo, uint64_t hi, int nowners,
                             uint32_t *const *slices, uint64_t slice_nodes, unsigned long long *probes,
                             void *stream);
/* Slices another process can map (one process per GPU, torch.distributed):
 * parba_ipc_alloc = cudaMalloc on the current device + cudaIpcGetMemHandle
 * (handle64: 64 bytes to send to the peers); parba_ipc_open maps a peer's
 * handle on the current device; parba_ipc_close / parba_ipc_free undo them. */
int parba_ipc_alloc(uint64_t bytes, void **dev_ptr, void *handle64);
/* 1 when kernels on `dev` can map `peer`'s memory and add into it with native
 * atomics (red.add over NVLink); routed counts need it of every pair. */
int parba_peer_atomics_ok(int dev, int peer);
int parba_ipc_open(const void *handle64, void **dev_ptr);
int parba_ipc_close(void *dev_ptr);
int parba_ipc_free(void *dev_ptr);

/* ---- Sequential-oracle counterpart (bb_generate, oracle.py:45-107) ------
 * The whole edge array E[0 .. 2m) (device, u64) built as an array: seed
 * cells, E[2i] = source(i), E[2i+1] = E[h(2i+1)] -- one hash per edge and
 * pointer jumping over the links, no hash chains (an independent check of
 * the tile kernels, as the reference's verify compares its parallel path
 * with the sequential fill, cli.py:332-351).  link: m - m0 u64 scratch;
 * flag: one device u32; *passes (optional) = pointer-jumping passes.
 * Plain mode (no option flags), uniform degree or degree sequence.
 * Synchronises `stream`. */
int parba_bb_fill(const parba_params_t *p, uint64_t *E, uint64_t *link, unsigned int *flag, int *passes,
                  void *stream);

/* ---- Remainder self-test (h % r, _kernels.py:32-42) --------------------
 * The exact-remainder routines of the tile kernels, callable on arbitrary
 * inputs so tests can pin them against integer division.  Methods: */
#define PARBA_MOD_FP31 0              /* r < 2^31 (chain values of 2-chunk launches) */
#define PARBA_MOD_FP_NARROW 1         /* r < 2^32                                  */
#define PARBA_MOD_FP_WIDE 2           /* r < 2^52 (4- and 5-chunk launches)         */
#define PARBA_MOD_INT 3               /* any r >= 1 (6 chunks, generic kernels)     */
#define PARBA_MOD_FP31_SERIES 4       /* the same three with 1/r from phase 1's     */
#define PARBA_MOD_FP_NARROW_SERIES 5  /* per-tile reciprocal series (r >= 2^27 + 224) */
#define PARBA_MOD_FP_WIDE_SERIES 6
#define PARBA_MOD_FP31_SERIES1 7      /* the series + one-stage remainder, r in [2^28 + 224, 2^31) */
#define PARBA_MOD_FP_WIDE_SERIES1 8   /* the same in 64 bits, r in [2^28 + 224, 2^52)              */
#define PARBA_MOD_FP32 9              /* r <= 0xF0000000 (chain values of 3-chunk launches): 32-bit tail */
#define PARBA_MOD_FP32_SERIES 10      /* the same with the series reciprocal                       */
/* out[k] = (hhi[k] * 2^32 + hlo[k]) mod r[k] by `method` (device buffers). */
int parba_debug_mod(int method, const uint32_t *hhi, const uint32_t *hlo, const uint64_t *r, uint64_t count,
                    uint64_t *out, void *stream);
/* `count` (h, r) pairs drawn on the device from `seed` (r log-uniform in
 * [rmin, rmax]; h uniform, next to a multiple of r, with an all-ones half,
 * or below 2r), each compared with exact u64 %: *mismatches += failures,
 * first_bad[0..2] = (h, r, result) of one failure.  Device buffers. */
int parba_debug_mod_check(int method, uint64_t seed, uint64_t count, uint64_t rmin, uint64_t rmax,
                          unsigned long long *mismatches, unsigned long long *first_bad, void *stream);
/* Exact relative-error bound of rcp.approx.ftz.f64 (it reads only the high
 * word of its operand, so 2^21 operands per exponent cover it): out[0] =
 * max |y0*x - 1| over biased exponents [e0, e0+ne), out[1] = the same after
 * the Newton step of the tile kernels' recip_approx.  Device buffer of 2
 * doubles. */
int parba_debug_rcp_bound(int e0, int ne, double *out, void *stream);

/* ---- Roofline denominators (measured next to the kernels, bench.py) ----
 * parba_peak_int32: launch an INT32 issue-rate kernel (LOP3 + IADD3 chains)
 * on `stream`; *lane_ops = the lane-operations it executes (time it with
 * events around the call).  scratch: one device u32.
 * parba_peak_write: 32-byte stores over buf[0, bytes) from many CTAs
 * (write-only HBM bandwidth; buf 32-byte aligned). */
int parba_peak_int32(uint32_t *scratch, double *lane_ops, void *stream);
int parba_peak_write(void *buf, uint64_t bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PARBA_B200_H */
