// parba_host.cu -- host-buffer entry points of the C ABI (blocking; the
// device generates in chunks while earlier chunks stream back) and the
// single-process multi-GPU driver parba_multi_run.
#include <cuda_runtime.h>

#include <emmintrin.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/vfs.h>
#include <unistd.h>
#include <cerrno>
#include <cstring>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/parba_b200.h"
#include "parba_common.h"

using namespace parba;
using namespace parba::host;

extern "C" {

// ---------------------------------------------------------------------------
// Host-buffer entry points.

namespace {

// Upload the host seed array; returns a params copy pointing at device memory.
int upload_seed(const parba_params_t *ph, parba_params_t *pd, DevBuf &seed) {
    *pd = *ph;
    if (ph->m0 > 0) {
        if (!ph->seed_edges) return fail(PARBA_EINVAL, "m0 > 0 but seed_edges is NULL");
        const size_t bytes = 2 * ph->m0 * sizeof(uint64_t);
        CUDA_TRY(cudaMalloc(&seed.p, bytes));
        CUDA_TRY(cudaMemcpy(seed.p, ph->seed_edges, bytes, cudaMemcpyHostToDevice));
        pd->seed_edges = (const uint64_t *)seed.p;
    }
    return PARBA_OK;
}


int generate_host_impl(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                       uint64_t *probes_host, int device, float *ms);

}  // namespace

int parba_generate_host(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                        uint64_t *probes_host, int device) {
    return generate_host_impl(ph, lo, hi, out_host, probes_host, device, nullptr);
}

namespace {
// pwrite every byte of [buf, buf + len) at `off` (cli.py:109-118)
int pwrite_all(int fd, const char *buf, uint64_t len, uint64_t off) {
    while (len) {
        const ssize_t k = pwrite(fd, buf, len, (off_t)off);
        if (k < 0) {
            if (errno == EINTR) continue;
            return fail(PARBA_EINVAL, "write failed at byte offset %llu: %s", (unsigned long long)off,
                        strerror(errno));
        }
        buf += k;
        off += (uint64_t)k;
        len -= (uint64_t)k;
    }
    return PARBA_OK;
}

// Files not in memory (a disk file system): rows generated into host
// buffers of 2^23 edges by the host pipeline while a writer thread pwrites
// the previous buffer (mapped writes there pay a page fault and a block
// allocation per page: 0.9 vs 2.4 GB/s measured into /tmp).
int write_binary_staged(const parba_params_t *ph, uint64_t lo, uint64_t hi, int fd, uint64_t off,
                        uint64_t *probes_host, int device) {
    constexpr uint64_t kChunk = 1ull << 23;
    const uint64_t C = hi - lo < kChunk ? hi - lo : kChunk;
    std::vector<uint64_t *> bufs(2, nullptr);
    for (auto &b : bufs)
        if (posix_memalign((void **)&b, 4096, C * 16) != 0) {
            for (auto &x : bufs) free(x);
            return fail(PARBA_EINVAL, "out of host memory for the file staging buffers");
        }
    int rc = PARBA_OK, wrc = PARBA_OK;
    std::thread writer;
    uint64_t probes = 0;
    std::string werr;
    int k = 0;
    for (uint64_t a = lo; a < hi && !rc; a += C, k ^= 1) {
        const uint64_t b = hi - a < C ? hi : a + C;
        uint64_t pr = 0;
        rc = generate_host_impl(ph, a, b, bufs[k], &pr, device, nullptr);
        probes += pr;
        if (writer.joinable()) writer.join();
        if (wrc) break;
        if (rc) break;
        writer = std::thread([&, k, a, b] {
            wrc = pwrite_all(fd, reinterpret_cast<const char *>(bufs[k]), 16 * (b - a), off + 16 * (a - lo));
            if (wrc) werr = parba_last_error();
        });
    }
    if (writer.joinable()) writer.join();
    for (auto &x : bufs) free(x);
    if (!rc && wrc) rc = fail(wrc, "%s", werr.c_str());
    if (!rc && probes_host) *probes_host = probes;
    return rc;
}
}  // namespace

int parba_write_binary(const parba_params_t *ph, uint64_t lo, uint64_t hi, int fd, uint64_t base_edge,
                       uint64_t *probes_host, int device) {
    if (probes_host) *probes_host = 0;
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (!rc) rc = check_range(ph, lo, hi);
    if (rc) return rc;
    if (lo < base_edge) return fail(PARBA_EINVAL, "lo (%llu) is below the file's first edge (%llu)",
                                    (unsigned long long)lo, (unsigned long long)base_edge);
    if (hi == lo) return PARBA_OK;
    struct stat sb;
    if (fd < 0 || fstat(fd, &sb) != 0) return fail(PARBA_EINVAL, "bad file descriptor %d", fd);
    const uint64_t off = 16 * (lo - base_edge), len = 16 * (hi - lo);
    if ((uint64_t)sb.st_size < off + len)
        return fail(PARBA_EINVAL, "file has %lld bytes, the range needs %llu", (long long)sb.st_size,
                    (unsigned long long)(off + len));
    // memory file systems (tmpfs, ramfs): map the range and fill it in place
    // (7.3 vs 3.6 GB/s for one pwrite thread into /dev/shm); anything else:
    // staged buffers + pwrite.  PARBA_WRITER_MMAP=0/1 forces either.
    struct statfs fs;
    const char *wm = getenv("PARBA_WRITER_MMAP");
    const bool in_memory = fstatfs(fd, &fs) == 0 && (fs.f_type == 0x01021994 /* TMPFS_MAGIC */ ||
                                                     fs.f_type == 0x858458f6 /* RAMFS_MAGIC */);
    if (wm ? wm[0] != '1' : !in_memory) return write_binary_staged(ph, lo, hi, fd, off, probes_host, device);
    const uint64_t pg = (uint64_t)sysconf(_SC_PAGESIZE);
    const uint64_t moff = off / pg * pg, mlen = len + (off - moff);
    // (MAP_POPULATE measured slower: 2.6 GB/s, the kernel faults the pages in on one thread)
    void *map = mmap(nullptr, mlen, PROT_READ | PROT_WRITE, MAP_SHARED, fd, (off_t)moff);
    if (map == MAP_FAILED)  // e.g. a write-only descriptor: staged buffers + pwrite instead
        return write_binary_staged(ph, lo, hi, fd, off, probes_host, device);
    uint64_t *rows = reinterpret_cast<uint64_t *>(static_cast<char *>(map) + (off - moff));
    rc = generate_host_impl(ph, lo, hi, rows, probes_host, device, nullptr);
    if (munmap(map, mlen) != 0 && !rc) rc = fail(PARBA_ECUDA, "munmap failed: %s", strerror(errno));
    return rc;
}

namespace {

// generate_block into host memory on one device; *ms (optional) = time
// from the first launch to the last row in host memory.
int generate_host_pairs(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                        uint64_t *probes_host, int device, float *ms);
int generate_host_targets(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                          uint64_t *probes_host, int device, float *ms);

int generate_host_impl(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                       uint64_t *probes_host, int device, float *ms) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (!rc) rc = check_range(ph, lo, hi);
    if (rc) return rc;
    if (probes_host) *probes_host = 0;
    if (ms) *ms = 0.f;
    if (hi == lo) return PARBA_OK;
    if (!out_host) return fail(PARBA_EINVAL, "out_pairs_host is NULL");
    const char *mode = getenv("PARBA_HOST_PAIRS");  // A/B: 16-byte rows over PCIe
    if (targets_only_ok(ph) && !(mode && mode[0] == '1'))
        return generate_host_targets(ph, lo, hi, out_host, probes_host, device, ms);
    return generate_host_pairs(ph, lo, hi, out_host, probes_host, device, ms);
}

// ---- pairs pipeline (SIMPLE hash, option flags, n > 2^32): 16-byte rows
// generated on the device in chunks, copied straight into the caller's
// array while the next chunk is generated.  *ms = device time from the
// first launch to the last copy.
int generate_host_pairs(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                        uint64_t *probes_host, int device, float *ms) {
    CUDA_TRY(cudaSetDevice(device));
    parba_params_t pd;
    DevBuf seed, bufs, prb;
    int rc = upload_seed(ph, &pd, seed);
    if (rc) return rc;
    // Two chunk buffers: the kernel fills one while the other drains over PCIe.
    const uint64_t total = hi - lo;
    uint64_t chunk = total < (1ull << 25) ? total : (1ull << 25);  // 32 Mi edges = 512 MiB
    if (ph->flags && chunk < total) chunk = chunk / ph->d > 0 ? (chunk / ph->d) * ph->d : ph->d;  // node cuts
    const size_t cbytes = chunk * 16;
    CUDA_TRY(cudaMalloc(&bufs.p, 2 * cbytes));
    CUDA_TRY(cudaMalloc(&prb.p, sizeof(unsigned long long)));
    StreamGuard sc, sx;
    CUDA_TRY(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&sx.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaMemsetAsync(prb.p, 0, sizeof(unsigned long long), sc.s));
    EventGuard t0, t1;
    CUDA_TRY(cudaEventCreate(&t0.e));
    CUDA_TRY(cudaEventCreate(&t1.e));
    CUDA_TRY(cudaEventRecord(t0.e, sc.s));
    EventGuard made[2], drained[2];
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(cudaEventCreateWithFlags(&made[b].e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&drained[b].e, cudaEventDisableTiming));
    }
    uint64_t k = 0;
    for (uint64_t a = lo; a < hi; a += chunk, ++k) {
        const uint64_t b = a + chunk < hi ? a + chunk : hi;
        const int slot = (int)(k & 1);
        uint64_t *dbuf = (uint64_t *)((char *)bufs.p + slot * cbytes);
        if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(sc.s, drained[slot].e, 0));
        rc = parba_generate(&pd, a, b, dbuf, (unsigned long long *)prb.p, sc.s);
        if (rc) return rc;
        CUDA_TRY(cudaEventRecord(made[slot].e, sc.s));
        CUDA_TRY(cudaStreamWaitEvent(sx.s, made[slot].e, 0));
        CUDA_TRY(cudaMemcpyAsync(out_host + 2 * (a - lo), dbuf, (b - a) * 16, cudaMemcpyDeviceToHost, sx.s));
        CUDA_TRY(cudaEventRecord(drained[slot].e, sx.s));
    }
    CUDA_TRY(cudaEventRecord(t1.e, sx.s));
    unsigned long long pr = 0;
    CUDA_TRY(cudaStreamSynchronize(sc.s));
    CUDA_TRY(cudaMemcpy(&pr, prb.p, sizeof(pr), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaStreamSynchronize(sx.s));
    if (ms) CUDA_TRY(cudaEventElapsedTime(ms, t0.e, t1.e));
    if (probes_host) *probes_host = pr;
    return PARBA_OK;
}


// ---- targets-only pipeline: the device writes the u32 target of every edge
// (4 B instead of 16), the copy engine moves it into pinned staging, and a
// team of host threads expands each staged chunk into (source, target) rows
// of the caller's array -- the source is the closed form (i - m0) / d + n0
// (generator.py:163-169), counted up edge by edge, and the rows are written
// with 16-byte streaming stores.  GPU, PCIe and host memory overlap over a
// ring of staging slots.  Host memory traffic is the bound (per edge: 16 B of
// rows written + the 4 B target written by the DMA and read back,
// tools/host_probe.cu), so small chunks help: a staged chunk that the CPU
// reads while it is still in the last-level cache costs no DRAM traffic.
// Optionally (PARBA_E2E_ROWS_FRAC, pinned output only) the first part of the
// range goes over PCIe as finished 16-byte rows concurrently with the CPU's
// part; measured slower on this pool's hosts, so off by default.

struct PipeCfg {
    uint64_t chunk = 1ull << 20;  // edges per staged chunk (4 MiB of targets: stays in the LLC)
    int slots = 4;                // staging slots in flight
    double rows_frac = 0.0;       // share of the range sent as 16-byte rows (pinned output only)
};

PipeCfg pipe_cfg() {
    PipeCfg c;
    if (const char *e = getenv("PARBA_E2E_CHUNK_LOG2")) {
        const int b = atoi(e);
        if (b >= 16 && b <= 26) c.chunk = 1ull << b;
    }
    if (const char *e = getenv("PARBA_E2E_SLOTS")) {
        const int k = atoi(e);
        if (k >= 2 && k <= 64) c.slots = k;
    }
    // measured on the B200 hosts (tools/e2e_perf.py, profiles/r02_e2e_sweep.jsonl):
    // the rows split only adds PCIe + DMA traffic to the bound host memory
    c.rows_frac = 0.0;
    if (const char *e = getenv("PARBA_E2E_ROWS_FRAC")) c.rows_frac = atof(e);
    if (c.rows_frac < 0.0) c.rows_frac = 0.0;
    if (c.rows_frac > 1.0) c.rows_frac = 1.0;
    return c;
}

// Staging per device, kept for the life of the process (pinned allocation
// costs more than a chunk's work); one host-array call per device at a time.
struct Staging {
    std::mutex use;
    uint32_t *host = nullptr;  // slots * chunk u32, pinned
    size_t host_words = 0;
    uint32_t *dev = nullptr;   // 2 * chunk u32 on the device
    size_t dev_words = 0;
    uint64_t *rows = nullptr;  // 2 * kRowChunk 16-byte rows on the device (rows split)
};
constexpr uint64_t kRowChunk = 1ull << 24;

Staging &staging_for(int device) {
    static std::mutex mu;
    static std::map<int, Staging *> all;
    std::lock_guard<std::mutex> lk(mu);
    auto it = all.find(device);
    if (it == all.end()) it = all.emplace(device, new Staging).first;
    return *it->second;
}

int host_threads() {
    if (const char *e = getenv("PARBA_HOST_THREADS")) {
        const int t = atoi(e);
        if (t > 0) return t;
    }
    cpu_set_t cs;
    CPU_ZERO(&cs);
    int n = 0;
    if (sched_getaffinity(0, sizeof(cs), &cs) == 0) n = CPU_COUNT(&cs);
    if (n <= 0) n = (int)std::thread::hardware_concurrency();
    return n > 2 ? n - 1 : 1;  // one core for the thread driving the GPU
}

// rows[k] = ((i0 + k - m0) / d + n0, tgt[k]) for k in [a, b)
void expand_rows(uint64_t *rows, const uint32_t *tgt, uint64_t i0, uint64_t a, uint64_t b, const parba_params_t *p,
                 bool nt) {
    if (b <= a) return;
    const uint64_t e = i0 + a - p->m0;
    uint64_t src = e / p->d + p->n0, rem = e % p->d;
    const uint64_t d = p->d;
    if (nt) {
        __m128i *o = reinterpret_cast<__m128i *>(rows);
        for (uint64_t k = a; k < b; ++k) {
            _mm_stream_si128(o + k, _mm_set_epi64x((long long)tgt[k], (long long)src));
            if (++rem == d) {
                rem = 0;
                ++src;
            }
        }
        _mm_sfence();
    } else {
        for (uint64_t k = a; k < b; ++k) {
            rows[2 * k] = src;
            rows[2 * k + 1] = tgt[k];
            if (++rem == d) {
                rem = 0;
                ++src;
            }
        }
    }
}

bool is_pinned(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

int generate_host_targets(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t *out_host,
                          uint64_t *probes_host, int device, float *ms) {
    const auto w0 = std::chrono::steady_clock::now();
    CUDA_TRY(cudaSetDevice(device));
    const PipeCfg cfg = pipe_cfg();
    const uint64_t C = cfg.chunk;
    const int S = cfg.slots;
    Staging &sg = staging_for(device);
    std::lock_guard<std::mutex> use(sg.use);
    if (sg.host_words < (size_t)S * C) {
        if (sg.host) cudaFreeHost(sg.host);
        sg.host = nullptr;
        sg.host_words = 0;
        CUDA_TRY(cudaHostAlloc((void **)&sg.host, (size_t)S * C * 4, cudaHostAllocPortable));
        sg.host_words = (size_t)S * C;
    }
    if (sg.dev_words < 2 * C) {
        if (sg.dev) cudaFree(sg.dev);
        sg.dev = nullptr;
        sg.dev_words = 0;
        CUDA_TRY(cudaMalloc((void **)&sg.dev, 2 * C * 4));
        sg.dev_words = 2 * C;
    }
    parba_params_t pd;
    DevBuf seed, prb;
    int rc = upload_seed(ph, &pd, seed);
    if (rc) return rc;
    const DevParams dp = make_dev(&pd);
    CUDA_TRY(cudaMalloc(&prb.p, 2 * sizeof(unsigned long long)));
    unsigned long long *prb_t = (unsigned long long *)prb.p, *prb_r = prb_t + 1;
    StreamGuard sc, sx, sc2, sx2;
    CUDA_TRY(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&sx.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaMemsetAsync(prb.p, 0, 2 * sizeof(unsigned long long), sc.s));
    CUDA_TRY(cudaStreamSynchronize(sc.s));

    // the rows part [lo, mid): generated as 16-byte rows, DMA'd straight into
    // the (pinned) caller's array on its own streams, no host work
    uint64_t mid = lo;
    if (cfg.rows_frac > 0.0 && hi - lo >= 4 * C && is_pinned(out_host))
        mid = lo + (uint64_t)((double)(hi - lo) * cfg.rows_frac);
    if (mid > lo) {
        if (!sg.rows) CUDA_TRY(cudaMalloc((void **)&sg.rows, 2 * kRowChunk * 16));
        CUDA_TRY(cudaStreamCreateWithFlags(&sc2.s, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&sx2.s, cudaStreamNonBlocking));
    }
    std::vector<EventGuard> rmade(2), rcopied(2);
    for (int b = 0; b < 2 && mid > lo; ++b) {
        CUDA_TRY(cudaEventCreateWithFlags(&rmade[b].e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&rcopied[b].e, cudaEventDisableTiming));
    }
    {
        uint64_t k = 0;
        for (uint64_t a = lo; a < mid; a += kRowChunk, ++k) {
            const uint64_t b = std::min(a + kRowChunk, mid);
            const int j = (int)(k & 1);
            uint64_t *dbuf = sg.rows + (uint64_t)j * 2 * kRowChunk;
            if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(sc2.s, rcopied[j].e, 0));
            if ((rc = launch_store(&pd, dp, a, b, dbuf, prb_r, sc2.s))) return rc;
            CUDA_TRY(cudaEventRecord(rmade[j].e, sc2.s));
            CUDA_TRY(cudaStreamWaitEvent(sx2.s, rmade[j].e, 0));
            CUDA_TRY(cudaMemcpyAsync(out_host + 2 * (a - lo), dbuf, (b - a) * 16, cudaMemcpyDeviceToHost, sx2.s));
            CUDA_TRY(cudaEventRecord(rcopied[j].e, sx2.s));
        }
    }

    // the targets part [mid, hi)
    std::vector<EventGuard> made(2), copied(S);
    for (auto &e : made) CUDA_TRY(cudaEventCreateWithFlags(&e.e, cudaEventDisableTiming));
    for (auto &e : copied) CUDA_TRY(cudaEventCreateWithFlags(&e.e, cudaEventDisableTiming));
    const int64_t nchunks = (int64_t)((hi - mid + C - 1) / C);
    const bool nt = (((uintptr_t)out_host) & 15) == 0;
    auto chunk_lo = [&](int64_t k) { return mid + (uint64_t)k * C; };
    auto chunk_n = [&](int64_t k) { return std::min(C, hi - chunk_lo(k)); };

    // GPU side of chunk k: targets into device buffer k % 2, then into slot k % S
    auto enqueue = [&](int64_t k) -> int {
        const int d = (int)(k & 1), s = (int)(k % S);
        uint32_t *dbuf = sg.dev + (uint64_t)d * C;
        if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(sc.s, copied[(k - 2) % S].e, 0));  // device buffer free
        int r = launch_store_t32(&pd, dp, chunk_lo(k), chunk_lo(k) + chunk_n(k), dbuf, prb_t, sc.s);
        if (r) return r;
        CUDA_TRY(cudaEventRecord(made[d].e, sc.s));
        CUDA_TRY(cudaStreamWaitEvent(sx.s, made[d].e, 0));
        CUDA_TRY(cudaMemcpyAsync(sg.host + (uint64_t)s * C, dbuf, chunk_n(k) * 4, cudaMemcpyDeviceToHost, sx.s));
        CUDA_TRY(cudaEventRecord(copied[s].e, sx.s));
        return PARBA_OK;
    };

    // host team: the staged chunks are cut into pieces of kPiece edges that
    // the workers claim in order from one atomic cursor (a descheduled thread
    // delays one piece, not a whole chunk).  The main thread alone waits on
    // the copy engine (one event per chunk), publishes staged chunks, and
    // recycles a slot once all of its pieces are done.
    const int T = host_threads();
    constexpr uint64_t kPiece = 1ull << 16;
    const uint64_t P = (C + kPiece - 1) / kPiece;  // pieces per chunk (the last chunk may use fewer)
    std::mutex mu;
    std::condition_variable cv_work, cv_main;
    int64_t ready = 0;                    // chunks staged in host memory (guarded by mu)
    std::vector<uint64_t> done(S, 0);     // pieces finished of the slot's current chunk (mu)
    bool abort = false;                   // (mu)
    std::atomic<uint64_t> next{0};
    const uint64_t total_pieces = nchunks ? (uint64_t)(nchunks - 1) * P + (chunk_n(nchunks - 1) + kPiece - 1) / kPiece : 0;
    auto pieces_of = [&](int64_t k) { return (chunk_n(k) + kPiece - 1) / kPiece; };
    auto worker = [&]() {
        for (;;) {
            const uint64_t q = next.fetch_add(1, std::memory_order_relaxed);
            if (q >= total_pieces) return;
            const int64_t k = (int64_t)(q / P);
            const uint64_t j = q % P;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_work.wait(lk, [&] { return ready > k || abort; });
                if (abort) return;
            }
            const int s = (int)(k % S);
            const uint64_t a = j * kPiece, b = std::min(a + kPiece, chunk_n(k));
            expand_rows(out_host + 2 * (chunk_lo(k) - lo), sg.host + (uint64_t)s * C, chunk_lo(k), a, b, ph, nt);
            std::lock_guard<std::mutex> lk(mu);
            if (++done[s] == pieces_of(k)) cv_main.notify_one();
        }
    };
    for (int64_t k = 0; k < std::min<int64_t>(S, nchunks); ++k)
        if ((rc = enqueue(k))) return rc;
    std::vector<std::thread> team;
    for (int w = 0; w < T && nchunks > 0; ++w) team.emplace_back(worker);
    for (int64_t k = 0; k < nchunks && !rc; ++k) {
        if (cudaEventSynchronize(copied[k % S].e) != cudaSuccess) {
            rc = fail(PARBA_ECUDA, "waiting for staged chunk %lld failed", (long long)k);
            std::lock_guard<std::mutex> lk(mu);
            abort = true;
            cv_work.notify_all();
            break;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            ready = k + 1;
        }
        cv_work.notify_all();
        if (k >= 1) {  // chunk k-1's slot is next in line for chunk k-1+S
            const int s = (int)((k - 1) % S);
            std::unique_lock<std::mutex> lk(mu);
            cv_main.wait(lk, [&] { return done[s] == pieces_of(k - 1); });
            done[s] = 0;
            lk.unlock();
            if (k - 1 + S < nchunks && (rc = enqueue(k - 1 + S))) {
                std::lock_guard<std::mutex> lk2(mu);
                abort = true;
                cv_work.notify_all();
            }
        }
    }
    for (auto &t : team) t.join();
    if (rc) return rc;
    if (mid > lo) CUDA_TRY(cudaStreamSynchronize(sx2.s));
    unsigned long long pr[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(pr, prb.p, sizeof(pr), cudaMemcpyDeviceToHost, sc.s));
    CUDA_TRY(cudaStreamSynchronize(sc.s));
    CUDA_TRY(cudaStreamSynchronize(sx.s));
    if (probes_host) *probes_host = pr[0] + pr[1];
    if (ms) *ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - w0).count();
    return PARBA_OK;
}

}  // namespace

int parba_degree_window_host(const parba_params_t *ph, uint64_t lo, uint64_t hi, uint64_t K,
                             int64_t *counts_host, uint64_t *probes_host, int device) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (!rc) rc = check_range(ph, lo, hi);
    if (rc) return rc;
    if (probes_host) *probes_host = 0;
    if (K > 0 && !counts_host) return fail(PARBA_EINVAL, "counts_host is NULL");
    CUDA_TRY(cudaSetDevice(device));
    parba_params_t pd;
    DevBuf seed, cnt, prb;
    rc = upload_seed(ph, &pd, seed);
    if (rc) return rc;
    const size_t cbytes = (K ? K : 1) * sizeof(unsigned long long);
    CUDA_TRY(cudaMalloc(&cnt.p, cbytes));
    CUDA_TRY(cudaMalloc(&prb.p, sizeof(unsigned long long)));
    StreamGuard sc;
    CUDA_TRY(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaMemsetAsync(cnt.p, 0, cbytes, sc.s));
    CUDA_TRY(cudaMemsetAsync(prb.p, 0, sizeof(unsigned long long), sc.s));
    rc = parba_degree_window(&pd, lo, hi, K, (unsigned long long *)cnt.p, (unsigned long long *)prb.p, sc.s);
    if (rc) return rc;
    std::vector<unsigned long long> tmp(K ? K : 1);
    unsigned long long pr = 0;
    CUDA_TRY(cudaMemcpyAsync(tmp.data(), cnt.p, cbytes, cudaMemcpyDeviceToHost, sc.s));
    CUDA_TRY(cudaMemcpyAsync(&pr, prb.p, sizeof(pr), cudaMemcpyDeviceToHost, sc.s));
    CUDA_TRY(cudaStreamSynchronize(sc.s));
    for (uint64_t v = 0; v < K; ++v) counts_host[v] += (int64_t)tmp[v];
    if (probes_host) *probes_host = pr;
    return PARBA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Single-process multi-GPU driver (SURVEY.md 8b parba_multi_run; the fork
// workers + Consumer.merge of driver.py:210-270 / analytics.py:78-82).
//
// Shards are contiguous edge ranges, each bound to a device.  One host thread
// per distinct device runs that device's shards back to back on one stream,
// accumulating degree counts into ONE device histogram (counts are +=), so a
// device that appears several times costs no extra reduction.  The distinct
// devices' histograms are then summed by one NCCL reduce (SUM, root = the
// first device) over NVLink -- the only collective on this path -- and the
// root's histogram is added into the caller's host array.  NCCL is loaded at
// run time (dlopen: the copy torch already loaded, else the system one), so
// the library has no link-time NCCL dependency.

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

namespace {

struct NcclApi {
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclReduce) reduce = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclGetVersion) get_version = nullptr;
    std::string why;  // non-empty when NCCL could not be loaded
};

const NcclApi &nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {getenv("PARBA_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        void *h = nullptr;
        for (const char *nm : names)  // a copy already in the process (torch's) first
            if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD))) break;
        for (const char *nm : names)
            if (!h && nm) h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char *e = dlerror();
            api.why = e ? e : "libnccl.so.2 not found";
            return;
        }
        api.init_all = (decltype(api.init_all))dlsym(h, "ncclCommInitAll");
        api.reduce = (decltype(api.reduce))dlsym(h, "ncclReduce");
        api.group_start = (decltype(api.group_start))dlsym(h, "ncclGroupStart");
        api.group_end = (decltype(api.group_end))dlsym(h, "ncclGroupEnd");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.get_version = (decltype(api.get_version))dlsym(h, "ncclGetVersion");
        if (!api.init_all || !api.reduce || !api.group_start || !api.group_end || !api.error_string)
            api.why = "libnccl is missing ncclCommInitAll / ncclReduce / ncclGroupStart / ncclGroupEnd";
    });
    return api;
}

#define NCCL_TRY(api, expr)                                                                              \
    do {                                                                                                 \
        ncclResult_t r_ = (expr);                                                                        \
        if (r_ != ncclSuccess) return fail(PARBA_ECUDA, "%s failed: %s", #expr, (api).error_string(r_)); \
    } while (0)

// One communicator clique per distinct device list, created once per process
// (ncclCommInitAll costs 0.1-1 s); a mutex per clique serialises its use.
struct Clique {
    std::vector<ncclComm_t> comms;
    std::mutex use;
};

int get_clique(const std::vector<int> &devs, Clique **out) {
    static std::mutex mu;
    static std::map<std::vector<int>, Clique *> cache;
    const NcclApi &api = nccl_api();
    if (!api.why.empty()) return fail(PARBA_ECUDA, "NCCL unavailable: %s", api.why.c_str());
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(devs);
    if (it == cache.end()) {
        auto *c = new Clique;
        c->comms.resize(devs.size());
        ncclResult_t r = api.init_all(c->comms.data(), (int)devs.size(), devs.data());
        if (r != ncclSuccess) {
            delete c;
            return fail(PARBA_ECUDA, "ncclCommInitAll(%zu devices) failed: %s", devs.size(), api.error_string(r));
        }
        it = cache.emplace(devs, c).first;  // kept for the life of the process
    }
    *out = it->second;
    return PARBA_OK;
}

// All shards of one distinct device.
struct DeviceRun {
    int dev = 0;
    std::vector<int> shards;  // indices into the caller's shard arrays
    int rc = PARBA_OK;
    std::string err;
    void *counts = nullptr;         // this device's histogram (count modes)
    unsigned long long *prb = nullptr;  // one probe counter per shard
    cudaStream_t st = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    float ms = 0.f;  // store mode: summed generate_host_impl device time
    DevBuf seed;     // seed graph on this device (alive until the run ends)
    // owner-routed full histogram: the slices this device owns (index into the
    // run's owner list) and the event recorded after they were zeroed
    std::vector<int> owned;
    cudaEvent_t zeroed = nullptr;
    DeviceRun() = default;
    DeviceRun(const DeviceRun &) = delete;
    DeviceRun &operator=(const DeviceRun &) = delete;
    ~DeviceRun() {
        if (counts || prb || st || t0 || t1 || seed.p) cudaSetDevice(dev);
        if (counts) cudaFree(counts);
        if (prb) cudaFree(prb);
        if (t0) cudaEventDestroy(t0);
        if (t1) cudaEventDestroy(t1);
        if (zeroed) cudaEventDestroy(zeroed);
        if (st) cudaStreamDestroy(st);
    }
};

// Owner-routed full histogram of one multi-device run: owner k holds nodes
// [k * slice, (k + 1) * slice) on device dev[k] (parba_degree_full_routed).
struct RoutedRun {
    std::vector<uint32_t *> ptr;  // one allocation per owner
    std::vector<int> dev;
    uint64_t slice = 0;
    ~RoutedRun() {
        for (size_t k = 0; k < ptr.size(); ++k)
            if (ptr[k]) {
                cudaSetDevice(dev[k]);
                cudaFree(ptr[k]);
            }
    }
};

// Every device of the run can map every other one's memory (enabled here)
// and add into it with native atomics (NVLink; not every PCIe path).
bool peers_ok(const std::vector<int> &udev) {
    for (int a : udev)
        for (int b : udev) {
            if (a == b) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) return false;
            if (!parba_peer_atomics_ok(a, b)) return false;
        }
    for (int a : udev) {
        if (cudaSetDevice(a) != cudaSuccess) return false;
        for (int b : udev) {
            if (a == b) continue;
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return false;
        }
    }
    return true;
}

size_t count_bytes(const parba_params_t *ph, int mode, uint64_t K) {
    return mode == PARBA_MULTI_FULL ? (size_t)ph->n * 4 : (size_t)(K ? K : 1) * 8;
}

// Run every shard of `r` on its device; counts stay on the device.
int run_device(const parba_params_t *ph, int mode, uint64_t K, const uint64_t *los, const uint64_t *his,
               void *out_host, uint64_t *shard_probes, DeviceRun &r, const RoutedRun *routed = nullptr,
               const std::vector<DeviceRun> *all = nullptr) {
    if (mode == PARBA_MULTI_STORE) {
        for (int s : r.shards) {
            float ms = 0.f;
            uint64_t pr = 0;
            int rc = generate_host_impl(ph, los[s], his[s], (uint64_t *)out_host + 2 * (los[s] - ph->m0), &pr,
                                        r.dev, &ms);
            if (rc) return rc;
            shard_probes[s] = pr;
            r.ms += ms;
        }
        return PARBA_OK;
    }
    CUDA_TRY(cudaSetDevice(r.dev));
    parba_params_t pd;
    int rc = upload_seed(ph, &pd, r.seed);
    if (rc) return rc;
    CUDA_TRY(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreate(&r.t0));
    CUDA_TRY(cudaEventCreate(&r.t1));
    const size_t ns = r.shards.size();
    CUDA_TRY(cudaMalloc((void **)&r.prb, ns * 8));
    CUDA_TRY(cudaMemsetAsync(r.prb, 0, ns * 8, r.st));
    const bool counted = mode != PARBA_MULTI_DISCARD && (mode == PARBA_MULTI_FULL || K > 0);
    if (routed) {
        // the slices this device owns were zeroed on its stream (event
        // `zeroed`, recorded before the worker threads started): wait for
        // every owner's, then count straight into the owners' slices
        for (const DeviceRun &o : *all) CUDA_TRY(cudaStreamWaitEvent(r.st, o.zeroed, 0));
        CUDA_TRY(cudaEventRecord(r.t0, r.st));
        for (size_t j = 0; j < ns; ++j) {
            const int s = r.shards[j];
            rc = parba_degree_full_routed(&pd, los[s], his[s], (int)routed->ptr.size(), routed->ptr.data(),
                                          routed->slice, r.prb + j, r.st);
            if (rc) return rc;
        }
        return PARBA_OK;
    }
    if (counted) {
        const size_t bytes = count_bytes(ph, mode, K);
        if (cudaMalloc(&r.counts, bytes) != cudaSuccess)
            return fail(PARBA_ENOMEM, "count buffer of %zu bytes on device %d", bytes, r.dev);
        CUDA_TRY(cudaMemsetAsync(r.counts, 0, bytes, r.st));
    }
    CUDA_TRY(cudaEventRecord(r.t0, r.st));
    for (size_t j = 0; j < ns; ++j) {
        const int s = r.shards[j];
        if (mode == PARBA_MULTI_FULL)
            rc = parba_degree_full(&pd, los[s], his[s], (uint32_t *)r.counts, r.prb + j, r.st);
        else
            rc = parba_degree_window(&pd, los[s], his[s], counted ? K : 0, (unsigned long long *)r.counts,
                                     r.prb + j, r.st);
        if (rc) return rc;
    }
    return PARBA_OK;  // probes are read after the reduction
}

template <typename T>
void add_into(int64_t *out, const std::vector<T> &x, uint64_t n) {
    for (uint64_t v = 0; v < n; ++v) out[v] += (int64_t)x[v];
}

}  // namespace

extern "C" {

int parba_multi_run_shards(const parba_params_t *ph, int nshards, const int *devs, const uint64_t *los,
                           const uint64_t *his, int mode, uint64_t K, void *out_host, uint64_t *probes_per_shard,
                           double *device_seconds) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (rc) return rc;
    if (nshards < 1 || !devs || !los || !his) return fail(PARBA_EINVAL, "need nshards >= 1 shards with devices");
    if (mode < PARBA_MULTI_STORE || mode > PARBA_MULTI_DISCARD) return fail(PARBA_EINVAL, "unknown mode %d", mode);
    if (mode == PARBA_MULTI_FULL) K = ph->n;
    if (!out_host && (mode == PARBA_MULTI_STORE || ((mode == PARBA_MULTI_WINDOW || mode == PARBA_MULTI_FULL) && K)))
        return fail(PARBA_EINVAL, "out_host is NULL");
    if (mode == PARBA_MULTI_FULL && 2 * (unsigned __int128)ph->m >= ((unsigned __int128)1 << 32))
        return fail(PARBA_EINVAL, "full histogram needs 2m < 2^32 (uint32 counters); use the window mode");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    for (int s = 0; s < nshards; ++s)
        if ((rc = check_range(ph, los[s], his[s]))) return rc;
    for (int s = 0; s < nshards; ++s)
        if (devs[s] < 0 || devs[s] >= ndev) return fail(PARBA_EINVAL, "device %d of shard %d not visible", devs[s], s);
    // group shards by distinct device, in order of first appearance
    std::vector<int> udev;
    for (int s = 0; s < nshards; ++s)
        if (std::find(udev.begin(), udev.end(), devs[s]) == udev.end()) udev.push_back(devs[s]);
    std::vector<DeviceRun> runs(udev.size());  // never resized: DeviceRun owns device memory
    for (int s = 0; s < nshards; ++s) {
        const size_t g = (size_t)(std::find(udev.begin(), udev.end(), devs[s]) - udev.begin());
        runs[g].dev = devs[s];
        runs[g].shards.push_back(s);
    }
    std::vector<uint64_t> probes(nshards, 0);
    // Full histogram on several devices with peer access: owner-routed counts
    // (the reduce fused into the count kernels) when the path applies to
    // every non-empty shard.  PARBA_MULTI_ROUTED: 0 = keep the ncclReduce, 1 =
    // routed even on one device; PARBA_MULTI_OWNERS = k: at least k owner
    // slices, dealt round-robin over the devices (tests of the routing).
    RoutedRun routed;
    bool use_routed = false;
    if (mode == PARBA_MULTI_FULL) {
        const char *e = getenv("PARBA_MULTI_ROUTED");
        const bool off = e && e[0] == '0', force = e && e[0] == '1';
        use_routed = !off && (runs.size() > 1 || force) && ph->n < (1ull << 32);
        for (int s = 0; use_routed && s < nshards; ++s)
            if (his[s] > los[s] && !parba_degree_full_routed_ok(ph, los[s], his[s])) use_routed = false;
        if (use_routed && runs.size() > 1 && !peers_ok(udev)) use_routed = false;
    }
    if (use_routed) {
        size_t owners = runs.size();
        if (const char *e = getenv("PARBA_MULTI_OWNERS")) owners = std::max(owners, (size_t)atoi(e));
        if (owners > 16) owners = 16;
        routed.slice = ((ph->n + owners - 1) / owners + 0xffffull) & ~0xffffull;
        routed.ptr.assign(owners, nullptr);
        routed.dev.assign(owners, 0);
        for (size_t k = 0; k < owners; ++k) {
            DeviceRun &r = runs[k % runs.size()];
            routed.dev[k] = r.dev;
            r.owned.push_back((int)k);
        }
        for (auto &r : runs) {
            CUDA_TRY(cudaSetDevice(r.dev));
            for (int k : r.owned) {
                if (cudaMalloc((void **)&routed.ptr[k], routed.slice * 4) != cudaSuccess)
                    return fail(PARBA_ENOMEM, "owner slice of %llu bytes on device %d",
                                (unsigned long long)routed.slice * 4, r.dev);
                CUDA_TRY(cudaMemsetAsync(routed.ptr[k], 0, routed.slice * 4, 0));
            }
            CUDA_TRY(cudaEventCreateWithFlags(&r.zeroed, cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(r.zeroed, 0));
        }
    }
    {
        std::vector<std::thread> th;
        for (auto &r : runs)
            th.emplace_back([&, rp = &r] {
                rp->rc = run_device(ph, mode, K, los, his, out_host, probes.data(), *rp,
                                    use_routed ? &routed : nullptr, &runs);
                if (rp->rc) rp->err = g_err;
            });
        for (auto &t : th) t.join();
    }
    for (auto &r : runs)
        if (r.rc) return fail(r.rc, "device %d: %s", r.dev, r.err.c_str());
    double secs = 0.0;
    if (mode == PARBA_MULTI_STORE) {
        for (auto &r : runs) secs = std::max(secs, (double)r.ms / 1000.0);
    } else if (use_routed) {
        for (auto &r : runs) {
            CUDA_TRY(cudaSetDevice(r.dev));
            CUDA_TRY(cudaEventRecord(r.t1, r.st));
        }
        for (auto &r : runs) {  // every stream drained: the owners' slices are complete
            CUDA_TRY(cudaSetDevice(r.dev));
            CUDA_TRY(cudaStreamSynchronize(r.st));
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, r.t0, r.t1));
            secs = std::max(secs, (double)ms / 1000.0);
            std::vector<unsigned long long> pr(r.shards.size());
            CUDA_TRY(cudaMemcpy(pr.data(), r.prb, pr.size() * 8, cudaMemcpyDeviceToHost));
            for (size_t j = 0; j < pr.size(); ++j) probes[r.shards[j]] = pr[j];
        }
        // every device copies its own slices to the host (one thread per
        // device: the copies run on all PCIe links at once)
        std::vector<std::thread> th;
        std::vector<int> rcs(runs.size(), PARBA_OK);
        for (size_t g = 0; g < runs.size(); ++g)
            th.emplace_back([&, g] {
                DeviceRun &r = runs[g];
                if (cudaSetDevice(r.dev) != cudaSuccess) {
                    rcs[g] = PARBA_ECUDA;
                    return;
                }
                for (int k : r.owned) {
                    const uint64_t v0 = (uint64_t)k * routed.slice;
                    if (v0 >= ph->n) continue;
                    const uint64_t cnt = std::min<uint64_t>(routed.slice, ph->n - v0);
                    std::vector<uint32_t> tmp(cnt);
                    if (cudaMemcpy(tmp.data(), routed.ptr[k], cnt * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
                        rcs[g] = PARBA_ECUDA;
                        return;
                    }
                    add_into((int64_t *)out_host + v0, tmp, cnt);
                }
            });
        for (auto &t : th) t.join();
        for (int c : rcs)
            if (c) return fail(c, "copy of an owner slice to the host failed");
    } else {
        const bool counted = runs[0].counts != nullptr;
        const char *force = getenv("PARBA_MULTI_NCCL");  // tests: NCCL even for one device
        if (counted && (runs.size() > 1 || (force && force[0] == '1'))) {
            Clique *cq = nullptr;
            if ((rc = get_clique(udev, &cq))) return rc;
            const NcclApi &api = nccl_api();
            std::lock_guard<std::mutex> lk(cq->use);
            const size_t n = mode == PARBA_MULTI_FULL ? ph->n : K;
            const ncclDataType_t ty = mode == PARBA_MULTI_FULL ? ncclUint32 : ncclUint64;
            NCCL_TRY(api, api.group_start());
            for (size_t g = 0; g < runs.size(); ++g) {
                CUDA_TRY(cudaSetDevice(runs[g].dev));
                ncclResult_t r = api.reduce(runs[g].counts, runs[g].counts, n, ty, ncclSum, 0, cq->comms[g],
                                            runs[g].st);
                if (r != ncclSuccess) {
                    api.group_end();
                    return fail(PARBA_ECUDA, "ncclReduce failed: %s", api.error_string(r));
                }
            }
            NCCL_TRY(api, api.group_end());
        }
        for (auto &r : runs) {
            CUDA_TRY(cudaSetDevice(r.dev));
            CUDA_TRY(cudaEventRecord(r.t1, r.st));
        }
        for (auto &r : runs) {
            CUDA_TRY(cudaSetDevice(r.dev));
            CUDA_TRY(cudaStreamSynchronize(r.st));
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, r.t0, r.t1));
            secs = std::max(secs, (double)ms / 1000.0);
            std::vector<unsigned long long> pr(r.shards.size());
            CUDA_TRY(cudaMemcpy(pr.data(), r.prb, pr.size() * 8, cudaMemcpyDeviceToHost));
            for (size_t j = 0; j < pr.size(); ++j) probes[r.shards[j]] = pr[j];
        }
        if (counted) {  // the root's histogram (= the sum) into the caller's array
            DeviceRun &r0 = runs[0];
            CUDA_TRY(cudaSetDevice(r0.dev));
            if (mode == PARBA_MULTI_FULL) {
                std::vector<uint32_t> tmp(ph->n);
                CUDA_TRY(cudaMemcpy(tmp.data(), r0.counts, ph->n * 4, cudaMemcpyDeviceToHost));
                add_into((int64_t *)out_host, tmp, ph->n);
            } else {
                std::vector<unsigned long long> tmp(K);
                CUDA_TRY(cudaMemcpy(tmp.data(), r0.counts, K * 8, cudaMemcpyDeviceToHost));
                add_into((int64_t *)out_host, tmp, K);
            }
        }
    }
    if (probes_per_shard)
        for (int s = 0; s < nshards; ++s) probes_per_shard[s] = probes[s];
    if (device_seconds) *device_seconds = secs;
    return PARBA_OK;
}

// Owner slices shared between processes (one process per GPU): plain
// cudaMalloc memory (the IPC handle of a pooled or sub-allocated block would
// name the whole block) and its 64-byte handle.
int parba_ipc_alloc(uint64_t bytes, void **dev_ptr, void *handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    if (!dev_ptr || !handle64 || bytes == 0) return fail(PARBA_EINVAL, "ipc_alloc needs a size and two outputs");
    void *ptr = nullptr;
    if (cudaMalloc(&ptr, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(PARBA_ENOMEM, "owner slice of %llu bytes", (unsigned long long)bytes);
    }
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
    if (e != cudaSuccess) {
        cudaFree(ptr);
        return fail(PARBA_ECUDA, "cudaIpcGetMemHandle failed: %s", cudaGetErrorString(e));
    }
    memcpy(handle64, &h, 64);
    *dev_ptr = ptr;
    return PARBA_OK;
}

int parba_peer_atomics_ok(int dev, int peer) {
    if (dev == peer) return 1;
    int can = 0, native = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can) {
        cudaGetLastError();
        return 0;
    }
    if (cudaDeviceGetP2PAttribute(&native, cudaDevP2PAttrNativeAtomicSupported, dev, peer) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return native ? 1 : 0;
}

int parba_ipc_open(const void *handle64, void **dev_ptr) {
    if (!handle64 || !dev_ptr) return fail(PARBA_EINVAL, "ipc_open needs a handle and an output");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return PARBA_OK;
}

int parba_ipc_close(void *dev_ptr) {
    if (dev_ptr) CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return PARBA_OK;
}

int parba_ipc_free(void *dev_ptr) {
    if (dev_ptr) CUDA_TRY(cudaFree(dev_ptr));
    return PARBA_OK;
}

int parba_multi_run(const parba_params_t *ph, int ndev, const int *devs, int mode, uint64_t K, void *out_host,
                    uint64_t *probes_host, double *device_seconds) {
    if (ph && is_deg(ph)) return fail(PARBA_EINVAL, "host entry points take uniform-degree families only");
    int rc = validate(ph);
    if (rc) return rc;
    if (ndev < 1 || !devs) return fail(PARBA_EINVAL, "need ndev >= 1 devices");
    const uint64_t total = ph->m - ph->m0;
    std::vector<uint64_t> lo(ndev), hi(ndev), pr(ndev);
    for (int g = 0; g < ndev; ++g) {
        lo[g] = ph->m0 + (uint64_t)(((unsigned __int128)total * g) / ndev);
        hi[g] = ph->m0 + (uint64_t)(((unsigned __int128)total * (g + 1)) / ndev);
        if (ph->flags) {  // node-granular: cut at node boundaries (uniform d)
            if (g > 0) lo[g] = node_first_edge(ph, ph->n0 + (lo[g] - ph->m0) / ph->d);
            if (g < ndev - 1) hi[g] = node_first_edge(ph, ph->n0 + (hi[g] - ph->m0) / ph->d);
        }
    }
    rc = parba_multi_run_shards(ph, ndev, devs, lo.data(), hi.data(), mode, K, out_host, pr.data(), device_seconds);
    if (rc) return rc;
    if (probes_host) {
        uint64_t s = 0;
        for (uint64_t x : pr) s += x;
        *probes_host = s;
    }
    return PARBA_OK;
}

}  // extern "C"
