/*
 * parba_oracle.c -- CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the CPU
 * baseline arm of bench.py).  Nothing in the product package
 * (paper_1602_07106_b200/) may link, load or call it; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * do.  It restates, in plain C, the algorithm of the reference package
 * `parba` (arXiv 1602.07106, Sanders & Schulz) exactly as the reference code
 * computes it -- table-driven CRC32-C with two accumulations per probe and a
 * hardware 64-bit remainder -- so its outputs are the reference's outputs.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function here
 * against the reference's own golden vectors (tests/helpers.py:11-18 of the
 * reference, frozen hash/chain values in its test_hashing.py / test_generator.py)
 * and against fixtures produced by importing the reference itself
 * (tests/golden/make_golden.py, fixtures in tests/golden/).
 *
 * Citations are to /root/reference/pkg/src/parba/<file>:<line>.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define PO_MASK32 0xFFFFFFFFull

/* hashing.py:40 -- reflected Castagnoli polynomial. */
#define PO_CRC32C_POLY 0x82F63B78u
/* hashing.py:36-37 -- salt-folding constants. */
#define PO_GOLDEN32 0x9E3779B9ull
#define PO_GOLDEN64 0x9E3779B97F4A7C15ull

enum { PO_KIND_CRC = 0, PO_KIND_SIMPLE = 1 };

typedef struct {
    uint64_t n, d, n0, m0, m;
    uint32_t kind;       /* PO_KIND_* */
    uint32_t s0, s1;     /* effective CRC seeds (HashConfig.crc_seeds) */
    uint64_t mult;       /* effective SIMPLE multiplier */
    const uint64_t *seed_edges; /* 2*m0 node IDs (may be NULL when m0 == 0) */
    /* degree sequence (generator.py:54-91, degreeseq.py:87-115): W[k] =
     * first edge of node n0+k, k <= n-n0 (W[n-n0] = m); NULL = uniform d */
    const uint64_t *W;
    /* option flags (generator.py:61-62): bit 0 no_self_loops, bit 1
     * no_parallel_edges; retry cap (0 = 64 * degree, generator.py:205) */
    uint32_t flags, pad;
    uint64_t max_attempts;
    /* raw HashConfig seed0 / seed1 / multiplier: retry attempt a >= 1 uses
     * the family with attempt_salt = a (HashConfig.with_attempt, hashing.py:69-71) */
    uint64_t base_seed0, base_seed1, base_mult;
} po_params_t;

static uint32_t g_table[256];
static int g_table_ready = 0;

/* hashing.py:88-95 -- bytewise reflected table. */
static void po_build_table(void) {
    if (g_table_ready) return;
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? ((c >> 1) ^ PO_CRC32C_POLY) : (c >> 1);
        g_table[i] = c;
    }
    g_table_ready = 1;
}

void po_crc32c_table(uint32_t out[256]) {
    po_build_table();
    memcpy(out, g_table, sizeof(g_table));
}

/* hashing.py:73-77 -- effective 32-bit seeds with the attempt salt folded in. */
void po_crc_seeds(uint64_t seed0, uint64_t seed1, uint64_t salt, uint32_t *s0, uint32_t *s1) {
    *s0 = (uint32_t)((seed0 + salt) & PO_MASK32);
    *s1 = (uint32_t)((seed1 + salt * PO_GOLDEN32) & PO_MASK32);
}

/* hashing.py:79-85 -- effective SIMPLE multiplier. */
uint64_t po_simple_multiplier(uint64_t multiplier, uint64_t salt) {
    return multiplier + 2ull * salt * PO_GOLDEN64; /* wraps mod 2^64 */
}

/* hashing.py:105-116 -- raw accumulator, 8 little-endian bytes, no inversion. */
uint32_t po_crc32c_u64(uint32_t seed, uint64_t word) {
    po_build_table();
    uint32_t c = seed;
    uint64_t w = word;
    for (int k = 0; k < 8; ++k) {
        c = g_table[(c ^ (uint32_t)w) & 0xFFu] ^ (c >> 8);
        w >>= 8;
    }
    return c;
}

/* _kernels.py:32-42 / hashing.py:119-125 -- ((crc(s0,r)<<32) + crc(s1,r)) % r.
 * r >= 1 is the caller's responsibility (the Python layer raises). */
static inline uint64_t po_h_crc_fast(uint64_t r, uint32_t s0, uint32_t s1) {
    uint32_t c0 = s0, c1 = s1;
    uint64_t w = r;
    for (int k = 0; k < 8; ++k) {
        uint32_t b = (uint32_t)(w & 0xFFu);
        c0 = g_table[(c0 & 0xFFu) ^ b] ^ (c0 >> 8);
        c1 = g_table[(c1 & 0xFFu) ^ b] ^ (c1 >> 8);
        w >>= 8;
    }
    uint64_t h = ((uint64_t)c0 << 32) + (uint64_t)c1;
    return h % r;
}

uint64_t po_h_crc(uint64_t r, uint32_t s0, uint32_t s1) {
    po_build_table();
    return po_h_crc_fast(r, s0, s1);
}

/* _kernels.py:20-29 / hashing.py:128-138 -- high 64 bits of ((r*M mod 2^64) * r). */
uint64_t po_h_simple(uint64_t r, uint64_t mult) {
    uint64_t t = r * mult;
    return (uint64_t)(((unsigned __int128)t * (unsigned __int128)r) >> 64);
}

static inline uint64_t po_hash(const po_params_t *p, uint64_t r) {
    return p->kind == PO_KIND_CRC ? po_h_crc_fast(r, p->s0, p->s1) : po_h_simple(r, p->mult);
}

/* generator.py:139-154, _kernels.py:45-75 -- walk r := h(r) (body at least
 * once) until r < stop_below or r is even.  Returns the probe count. */
static inline uint64_t po_chain(const po_params_t *p, uint64_t r, uint64_t stop_below, uint64_t *term) {
    uint64_t probes = 0;
    for (;;) {
        r = po_hash(p, r);
        ++probes;
        if (r < stop_below || (r & 1ull) == 0) break;
    }
    *term = r;
    return probes;
}

/* _kernels.py:121-135 -- resolve_chain_block: fresh output, r0 untouched. */
uint64_t po_resolve_chain_block(const po_params_t *p, const uint64_t *r0, uint64_t count,
                                uint64_t stop_below, uint64_t *out) {
    po_build_table();
    uint64_t probes = 0;
    for (uint64_t k = 0; k < count; ++k) probes += po_chain(p, r0[k], stop_below, &out[k]);
    return probes;
}

/* degreeseq.py:188-196 -- node_of_edge_bisect: the rightmost k with
 * W[k] <= e (zero-degree nodes share their successor's W and are skipped). */
static inline uint64_t po_node_bisect(const po_params_t *p, uint64_t e) {
    uint64_t lo = 0, hi = p->n - p->n0;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (p->W[mid] <= e) lo = mid + 1;
        else hi = mid;
    }
    return p->n0 + lo - 1;
}

/* generator.py:157-169 -- closed forms (uniform d) or owner lookup. */
static inline uint64_t po_source(const po_params_t *p, uint64_t i) {
    if (p->W) return po_node_bisect(p, i);
    return (i - p->m0) / p->d + p->n0;
}
static inline uint64_t po_target(const po_params_t *p, uint64_t term) {
    if (term < 2 * p->m0) return p->seed_edges[term];          /* generator.py:164-165, 312-318 */
    if (p->W) return po_node_bisect(p, term >> 1);              /* generator.py:168-169 */
    return ((term >> 1) - p->m0) / p->d + p->n0;                /* generator.py:166-168, 320-322 */
}

static inline uint64_t po_first_edge(const po_params_t *p, uint64_t v) {
    return p->W ? p->W[v - p->n0] : p->m0 + (v - p->n0) * p->d;
}
static inline uint64_t po_degree(const po_params_t *p, uint64_t v) {
    return p->W ? p->W[v - p->n0 + 1] - p->W[v - p->n0] : p->d;
}

/* hashing.py:69-85 -- the family of retry attempt a (a = 0: the configured one). */
static po_params_t po_family(const po_params_t *p, uint64_t attempt) {
    po_params_t f = *p;
    if (attempt) {
        po_crc_seeds(p->base_seed0, p->base_seed1, attempt, &f.s0, &f.s1);
        f.mult = po_simple_multiplier(p->base_mult, attempt);
    }
    return f;
}

/* generator.py:184-217 -- _node_edges_with_probes: node v's edges, in edge
 * order, into rows[dv][2].  Returns 0, or -1 with *fail_edge set when
 * no_parallel_edges finds no fresh target within the cap. */
int po_node_edges(const po_params_t *p, uint64_t v, uint64_t *rows, uint64_t *probes, uint64_t *fail_edge) {
    po_build_table();
    const uint64_t first = po_first_edge(p, v), dv = po_degree(p, v);
    const uint64_t stop = 2 * p->m0;
    const int nsl = p->flags & 1u, npe = (p->flags >> 1) & 1u;
    for (uint64_t i = first; i < first + dv; ++i) {
        const uint64_t r0 = nsl ? 2 * first : 2 * i + 1;
        uint64_t term, t = 0;
        if (!npe) {
            *probes += po_chain(p, r0, stop, &term);
            t = po_target(p, term);
        } else {
            const uint64_t cap = p->max_attempts ? p->max_attempts : 64 * dv;
            int fresh = 0;
            for (uint64_t a = 0; a < cap && !fresh; ++a) {
                const po_params_t f = po_family(p, a);
                *probes += po_chain(&f, r0, stop, &term);
                t = po_target(p, term);
                fresh = 1;
                for (uint64_t j = first; j < i; ++j)
                    if (rows[2 * (j - first) + 1] == t) { fresh = 0; break; }
            }
            if (!fresh) { *fail_edge = i; return -1; }
        }
        rows[2 * (i - first)] = v;
        rows[2 * (i - first) + 1] = t;
    }
    return 0;
}

/* generator.py:231-245 -- node whose first edge is exactly pos (n at m). */
static int po_boundary_node(const po_params_t *p, uint64_t pos, uint64_t *v) {
    if (pos == p->m) { *v = p->n; return 0; }
    uint64_t u = po_source(p, pos);
    if (po_first_edge(p, u) != pos) return -1;
    *v = u;
    return 0;
}

/* generator.py:258-302, flag modes -- node-granular generate_block.
 * Returns 0, 1 (lo or hi is not a node boundary), 2 (infeasible: *fail_edge). */
int po_generate_nodes(const po_params_t *p, uint64_t lo, uint64_t hi, uint64_t *out_pairs,
                      uint64_t *probes, uint64_t *fail_edge) {
    uint64_t vlo, vhi;
    *probes = 0;
    if (lo == hi) return 0;
    if (po_boundary_node(p, lo, &vlo) || po_boundary_node(p, hi, &vhi)) return 1;
    for (uint64_t v = vlo; v < vhi; ++v)
        if (po_node_edges(p, v, out_pairs + 2 * (po_first_edge(p, v) - lo), probes, fail_edge)) return 2;
    return 0;
}

/* generator.py:258-325 (plain path, uniform d) -- rows (src, tgt) of edges
 * lo..hi-1 into out_pairs[2*(hi-lo)].  Returns total probes. */
uint64_t po_generate_block(const po_params_t *p, uint64_t lo, uint64_t hi, uint64_t *out_pairs) {
    po_build_table();
    uint64_t probes = 0;
    const uint64_t stop = 2 * p->m0;
    for (uint64_t i = lo; i < hi; ++i) {
        uint64_t term;
        probes += po_chain(p, 2 * i + 1, stop, &term);  /* generator.py:302-304 */
        out_pairs[2 * (i - lo)] = po_source(p, i);
        out_pairs[2 * (i - lo) + 1] = po_target(p, term);
    }
    return probes;
}

/* analytics.py:44-48 -- both endpoints with id < K (self-loop counts 2). */
void po_count_block(const uint64_t *pairs, uint64_t nedges, int64_t *counts, uint64_t K) {
    for (uint64_t k = 0; k < 2 * nedges; ++k)
        if (pairs[k] < K) counts[pairs[k]] += 1;
}

/* generate_block + DegreeCountConsumer.accept_block (analytics.py:75-76),
 * edge by edge, without materialising the block.  Returns total probes. */
uint64_t po_degree_block(const po_params_t *p, uint64_t lo, uint64_t hi, uint64_t K, int64_t *counts) {
    po_build_table();
    uint64_t probes = 0;
    const uint64_t stop = 2 * p->m0;
    for (uint64_t i = lo; i < hi; ++i) {
        uint64_t term;
        probes += po_chain(p, 2 * i + 1, stop, &term);
        uint64_t s = po_source(p, i), t = po_target(p, term);
        if (s < K) counts[s] += 1;
        if (t < K) counts[t] += 1;
    }
    return probes;
}

/* oracle.py:101-106 -- derandomized sequential Batagelj-Brandes fill,
 * E[2i] = src(i); E[2i+1] = E[h(2i+1)].  e has 2*m entries. */
void po_bb_generate(const po_params_t *p, uint64_t *e) {
    po_build_table();
    for (uint64_t k = 0; k < 2 * p->m0; ++k) e[k] = p->seed_edges[k];
    for (uint64_t i = p->m0; i < p->m; ++i) {
        e[2 * i] = po_source(p, i);
        e[2 * i + 1] = e[po_hash(p, 2 * i + 1)];
    }
}

/* ------------------------------------------------------------------------
 * Threaded CPU baseline: the reference driver (driver.py:161-270) cuts
 * [lo,hi) into contiguous batches claimed from a shared cursor by W
 * workers; each batch runs generate_block and then the consumer.  Here the
 * workers are pthreads and the cursor an atomic counter.  mode 0: store
 * (pairs written to out_pairs at 2*(i-lo)); mode 1: degree window (private
 * int64[K] per worker, summed at the end, analytics.py:78-82); mode 2:
 * discard.  Returns total probes. */
typedef struct {
    const po_params_t *p;
    uint64_t lo, hi, batch, K;
    int mode;
    uint64_t *out_pairs;
    int64_t *counts;      /* merged result */
    uint64_t next;        /* shared cursor, batch index */
    pthread_mutex_t lock;
} po_run_t;

typedef struct { po_run_t *run; uint64_t probes; int64_t *ctx; } po_worker_t;

static void *po_worker_main(void *arg) {
    po_worker_t *w = (po_worker_t *)arg;
    po_run_t *R = w->run;
    uint64_t nb = (R->hi - R->lo + R->batch - 1) / R->batch;
    uint64_t *scratch = (R->mode == 0) ? NULL : (uint64_t *)malloc(2 * R->batch * sizeof(uint64_t));
    for (;;) {
        uint64_t k = __atomic_fetch_add(&R->next, 1, __ATOMIC_RELAXED);
        if (k >= nb) break;
        uint64_t a = R->lo + k * R->batch;
        uint64_t b = a + R->batch < R->hi ? a + R->batch : R->hi;
        if (R->mode == 0) {
            w->probes += po_generate_block(R->p, a, b, R->out_pairs + 2 * (a - R->lo));
        } else {
            w->probes += po_generate_block(R->p, a, b, scratch);
            if (R->mode == 1) po_count_block(scratch, b - a, w->ctx, R->K);
        }
    }
    free(scratch);
    return NULL;
}

uint64_t po_run_threaded(const po_params_t *p, uint64_t lo, uint64_t hi, int mode, uint64_t K,
                         int nthreads, uint64_t batch, uint64_t *out_pairs, int64_t *counts) {
    po_build_table();
    if (nthreads < 1) nthreads = 1;
    if (batch < 1) batch = 1 << 16;
    po_run_t R;
    memset(&R, 0, sizeof(R));
    R.p = p; R.lo = lo; R.hi = hi; R.batch = batch; R.K = K; R.mode = mode;
    R.out_pairs = out_pairs; R.counts = counts; R.next = 0;
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    po_worker_t *ws = (po_worker_t *)calloc((size_t)nthreads, sizeof(po_worker_t));
    for (int t = 0; t < nthreads; ++t) {
        ws[t].run = &R;
        ws[t].ctx = (mode == 1) ? (int64_t *)calloc(K ? K : 1, sizeof(int64_t)) : NULL;
        pthread_create(&th[t], NULL, po_worker_main, &ws[t]);
    }
    uint64_t probes = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        probes += ws[t].probes;
        if (mode == 1) {
            for (uint64_t v = 0; v < K; ++v) counts[v] += ws[t].ctx[v];
            free(ws[t].ctx);
        }
    }
    free(th);
    free(ws);
    return probes;
}
