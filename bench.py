#!/usr/bin/env python
"""Benchmark: edges generated / s (device-timed) for the Sanders-Schulz BA
generator on B200 -- BASELINE.json's metric on its configs[1] (store mode,
n=1e8, d=10, m=1e9 int64 pairs written to HBM), the fixed graph's edge-ID
range sharded over the GPUs as configs[1] prescribes (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL).

One JSON line on rank 0.  `value` = whole-job edges/s with the output
resident in HBM; `e2e` = the same metric through the reference-facing API
`generate_block(lo, hi, p)` returning a host array (its device->host traffic
inside the timed region); `roofline` = the store kernel's algorithmic
16 B/edge write rate against the measured HBM peak; `modes` = the streaming
configs (C3 window, C4 full histogram, C5 the paper's demo), each with its
own device time, NCCL reduce included, and an integer roofline against the
INT32 peak measured in the same run; `cpu_baseline` = the reference itself
(parba + numba from baseline/_ref) on all host cores, with the C port of the
oracle beside it.  `--impl reference` times the reference alone.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(n=10**8, d=10)          # configs[1]: store mode, m = 1e9
C3 = dict(n=10**9, d=100, K=10**5)  # configs[2]: streaming window, m = 1e11
C4 = dict(n=10**8, d=16)          # configs[3]: full histogram, m = 1.6e9
C5 = dict(n=10**10, d=100, K=10**5)  # configs[4]: the paper's demo, m = 1e12
METRIC = "edges generated/sec (device-timed) at 1/2/4/8 B200; % of HBM/int roofline"  # BASELINE.json metric
BYTES_PER_EDGE = 16               # algorithmic HBM bytes per stored edge
E2E_EDGES = 250_000_000  # edges per GPU returned to the host per e2e step (4 GB)
INT_OPS_PER_PROBE = 32            # SURVEY 8d convention (64 per edge)


def _peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every ~5 ms) DURING the
    timed region; falls back to nvidia-smi when NVML is unavailable."""

    def __init__(self, index: int, period: float = 0.005):
        self.index = index
        self.period = period
        self.sm: list[float] = []
        self.max_sm: float | None = None
        self.reasons: set[str] = set()
        self.n = 0
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                    "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                    "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            while True:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.reasons |= {k for k, b in bits.items() if r & b}
                self.n += 1
                if self._stop.wait(self.period):
                    break
        except Exception:
            Q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap"
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip().split(",")
                    self.sm.append(float(out[0]))
                    self.max_sm = float(out[1])
                    if out[2].strip() == "Active":
                        self.reasons.add("hw_slowdown")
                    if out[3].strip() == "Active":
                        self.reasons.add("sw_power_cap")
                    self.n += 1
                except Exception:
                    pass
                self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm,
                "reasons": sorted(self.reasons), "samples": self.n}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, ws, local


def cpu_baseline(sample_edges: int | None = None, budget_s: float = 12.0) -> dict:
    """The reference algorithm (C port in oracle/) on the host cores, store
    mode into host memory over a bounded sample of C2's edge range: chunks of
    at most 1e8 edges (1.6 GB buffer, reused) walking down from the top of
    the ID space until about `budget_s` of CPU work is done."""
    import numpy as np

    import oracle as O

    threads = len(os.sched_getaffinity(0))
    p = O.OParams(n=C2["n"], d=C2["d"])
    # calibrate on a small top-of-range sample, then size for ~budget_s
    t0 = time.perf_counter()
    O.run_threaded(p, p.m - 2_000_000, p.m, O.MODE_STORE, threads=threads, batch=1 << 16)
    rate = 2_000_000 / (time.perf_counter() - t0)
    if sample_edges is None:
        sample_edges = int(min(max(rate * budget_s, 4_000_000), p.m))
    chunk = min(sample_edges, 100_000_000)
    out = np.empty((chunk, 2), dtype=np.uint64)
    done = probes = 0
    hi = p.m
    t0 = time.perf_counter()
    while done < sample_edges:
        n = min(chunk, sample_edges - done)
        _, pr = O.run_threaded(p, hi - n, hi, O.MODE_STORE, threads=threads, batch=1 << 16, out=out[:n])
        probes += pr
        done += n
        hi -= n
    dt = time.perf_counter() - t0
    return {"value": sample_edges / dt, "unit": "edges/s", "cores": threads, "kind": "port",
            "sample": f"C2 (n=1e8, d=10) edge IDs [{p.m - sample_edges}, {p.m}) = {sample_edges} edges, "
                      f"store mode into a reused host buffer, oracle/parba_oracle.c (the reference's "
                      f"table CRC + u64 %), {threads} threads, {dt:.2f} s",
            "sample_edges": sample_edges, "probes_per_edge": probes / sample_edges}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_CFG = {"store": (C2["n"], C2["d"], 0), "window": (C3["n"], C3["d"], C3["K"]),
           "full": (C4["n"], C4["d"], C4["n"])}


def _ref_worker(args):
    """One forked worker of the reference's own driver loop (parba/driver.py
    _work_loop: claim a 2^16-edge batch, generate_block, accept_block)."""
    wid, mode, n, d, K, batches, cursor, out_q = args
    try:
        import parba.driver as rd
        from parba.analytics import DegreeCountConsumer
        from parba.generator import GenParams

        p = GenParams(n=n, d=d)
        consumer = rd.DiscardConsumer() if mode == "store" else DegreeCountConsumer(K)
        blist = [rd.Batch(a, b) for a, b in batches]

        def claim():
            with cursor.get_lock():
                k = cursor.value
                cursor.value = k + 1
                return k

        ctx, st = rd._work_loop(wid, p, consumer, blist, claim, None, "rank")
        out_q.put(("ok", wid, st.edges, st.probes, int(ctx.sum()) if mode != "store" else int(ctx)))
    except BaseException as e:  # surfaced by the parent
        out_q.put(("error", wid, repr(e), 0, 0))


def reference_numba(mode: str = "store", sample_edges: int | None = None, budget_s: float = 10.0,
                    threads: int | None = None) -> dict:
    """The reference itself (parba from baseline/_ref: numba kernels, its
    own generate_block / consumers / batch loop, fork workers like
    driver.run) on all host cores over the top `sample_edges` edge IDs of
    the config's range.  Returns a cpu_baseline dict (kind "reference")."""
    import multiprocessing as mp

    if not os.path.isdir(os.path.join(REF_DIR, "parba")):
        raise RuntimeError("baseline/_ref is not installed")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/parba_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import parba._kernels as rk
    from parba.generator import GenParams, generate_block

    rk.warmup()  # compile before the fork, as driver.run does
    threads = threads or len(os.sched_getaffinity(0))
    n, d, K = REF_CFG[mode]
    m = n * d
    bs = 1 << 16  # driver.DEFAULT_BATCH_SIZE
    if sample_edges is None:  # calibrate one core on the top of the range
        p = GenParams(n=n, d=d)
        t0 = time.perf_counter()
        for k in range(8):
            generate_block(m - (k + 1) * bs, m - k * bs, p)
        rate = 8 * bs / (time.perf_counter() - t0)
        sample_edges = int(min(m, max(rate * threads * budget_s, threads * bs)))
        sample_edges -= sample_edges % bs
    lo = m - sample_edges
    batches = [(a, min(a + bs, m)) for a in range(lo, m, bs)]
    ctx = mp.get_context("fork")
    cursor = ctx.Value("q", 0)
    out_q = ctx.Queue()
    t0 = time.perf_counter()
    procs = [ctx.Process(target=_ref_worker, args=((w, mode, n, d, K, batches, cursor, out_q),))
             for w in range(threads)]
    for pr in procs:
        pr.start()
    msgs = [out_q.get() for _ in procs]
    for pr in procs:
        pr.join()
    dt = time.perf_counter() - t0
    bad = [mm for mm in msgs if mm[0] != "ok"]
    if bad:
        raise RuntimeError(f"reference worker failed: {bad[0]}")
    edges = sum(mm[2] for mm in msgs)
    assert edges == sample_edges, (edges, sample_edges)
    what = {"store": "generate_block per 2^16-edge batch into fresh host arrays (DiscardConsumer)",
            "window": f"generate_block + count_block, K={K} (DegreeCountConsumer)",
            "full": "generate_block + count_block, K=n (DegreeCountConsumer)"}[mode]
    return {"value": sample_edges / dt, "unit": "edges/s", "cores": threads, "kind": "reference",
            "sample": f"the reference parba (baseline/_ref, numba {_numba_version()}) on edge IDs "
                      f"[{lo}, {m}) of n={n:.0e}, d={d}: {what}, its own batch loop "
                      f"(driver._work_loop) in {threads} forked workers, {dt:.2f} s",
            "sample_edges": sample_edges, "probes_per_edge": sum(mm[3] for mm in msgs) / sample_edges,
            "seconds": dt}


def _numba_version() -> str:
    try:
        import numba

        return numba.__version__
    except Exception:  # pragma: no cover
        return "?"


def c2_config(ws: int) -> dict:
    """The workload both arms report (BASELINE.json configs[1])."""
    m = C2["n"] * C2["d"]
    return {"workload": "configs[1]: store mode, n=1e8, d=10, m=1e9 edges -> (m,2) u64 pairs (16 GB) "
                        "in HBM, contiguous edge-ID shards over the GPUs (total work fixed)",
            "n": C2["n"], "d": C2["d"], "m": m, "shard_edges": m // ws,
            "parallelism": f"edge-range shards x{ws} (no collective in store mode)",
            "l2": "output 16 GB/N >> 126 MB L2: no flush needed between steps"}


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _relaunch(n: int) -> int:
    """bench.py --gpus N without a torchrun environment: run N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_reference(args) -> None:
    """The reference arm: parba itself (baseline/_ref, numba) on all host
    cores, store mode on C2, one bounded sample per step; rank 0 only."""
    rank, ws, _ = _dist()
    if rank != 0:
        return
    try:
        first = reference_numba("store", budget_s=3.0)
        measure = lambda n: reference_numba("store", sample_edges=n)  # noqa: E731
    except Exception as e:  # no baseline/_ref: the oracle's C port instead
        print(f"reference parba unavailable ({e!r}); timing the C port", file=sys.stderr)
        first = cpu_baseline(budget_s=3.0)
        measure = lambda n: cpu_baseline(sample_edges=n)  # noqa: E731
    n_edges = first["sample_edges"]
    samples = []
    for k in range(args.warmup + args.steps):
        cb = first if k == 0 else measure(n_edges)
        if k >= args.warmup:
            samples.append(cb)
    value = statistics.median(s["value"] for s in samples)
    line = {"impl": "reference", "metric": METRIC,
            "value": value, "unit": "edges/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * n_edges / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": c2_config(ws) | {"sample_edges": n_edges,
                                       "reference_step": "a bounded CPU sample of the workload per step"},
            "cpu_baseline": {k: samples[-1][k] for k in ("kind", "cores", "sample")} | {"value": value,
                                                                                        "unit": "edges/s"},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=9)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-modes", action="store_true")
    ap.add_argument("--profile", action="store_true", help="store kernel only (for ncu)")
    ap.add_argument("--only", default=None, help="one streaming mode only (window_c3|full_c4|window_c5), for ncu")
    ap.add_argument("--share-gpu", action="store_true",
                    help="control-flow check of the N-rank path on ONE GPU (gloo, every rank on cuda:0); "
                         "its numbers are not measurements")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not (args.profile or args.only) else args.warmup

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
        return

    rank, ws, local = _dist()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    # host threads of the e2e pipeline: this rank's share of the host cores
    lws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    ncpu = len(os.sched_getaffinity(0))
    os.environ.setdefault("PARBA_HOST_THREADS", str(max(1, ncpu // lws - 1 if ncpu // lws > 2 else 1)))
    # CPU baselines first (N=1, rank 0), before any CUDA work
    cpu = None
    if rank == 0 and ws == 1 and not (args.no_cpu_baseline or args.profile or args.only):
        port = cpu_baseline(budget_s=6.0)
        try:
            cpu = reference_numba("store", budget_s=8.0)
            cpu["port"] = {k: port[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # baseline/_ref missing
            cpu = port | {"reference_unavailable": repr(e)}

    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1602_07106_b200 as pb

    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L = pb._lib.load()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather(x: float) -> list[float]:
        if ws == 1:
            return [x]
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        out = [torch.zeros_like(t) for _ in range(ws)]
        dist.all_gather(out, t)
        return [float(o.item()) for o in out]

    def timed(fn, reps: int = 3) -> float:
        """best device time (s) of fn() over reps, CUDA events on `stream`."""
        best = 1e30
        for _ in range(reps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            best = min(best, a.elapsed_time(b) / 1000.0)
        return best

    # ---------------- store mode, C2 (headline): BASELINE.json configs[1] is
    # one fixed graph (n=1e8, d=10) "sharded by contiguous edge-ID ranges over
    # 1/2/4/8 GPUs", so total work is fixed as N grows (strong scaling).
    p = pb.GenParams(**C2)
    lo, hi = pb.parallel.shard_range(0, p.m, rank, ws)
    shard = hi - lo
    out = torch.empty((shard if not args.only else 1, 2), dtype=torch.int64, device=dev)
    probes = torch.zeros(1, dtype=torch.int64, device=dev)
    cp = p._device_params(dev)

    # roofline denominators measured here, on this GPU, before the kernels
    peaks = {}
    if not (args.profile or args.only):
        wsec = timed(lambda: pb._lib.check(L.parba_peak_write(out.data_ptr(), shard * 16, stream.cuda_stream)),
                     reps=5)
        fsec = timed(lambda: out.fill_(7), reps=5)  # torch's vectorised fill: another write-only kernel
        scratch = torch.zeros(1, dtype=torch.int32, device=dev)
        ops = ctypes.c_double(0.0)
        isec = timed(lambda: pb._lib.check(L.parba_peak_int32(scratch.data_ptr(), ctypes.byref(ops),
                                                              stream.cuda_stream)))
        peaks = {"write_only_gbs": shard * 16 / min(wsec, fsec) / 1e9, "int32_lane_ops_per_s": ops.value / isec,
                 "write_only_gbs_parba": shard * 16 / wsec / 1e9, "write_only_gbs_torch_fill": shard * 16 / fsec / 1e9,
                 "how": "in this run on this GPU: the faster of 32-byte stores over the store buffer from "
                        "148x32 CTAs (parba_peak_write) and torch's fill_ (best of 5 each); LOP3+IADD3 chains "
                        "(parba_peak_int32), best of 3"}

    def store_step():
        pb._lib.check(L.parba_generate(cp, lo, hi, out.data_ptr(), probes.data_ptr(), stream.cuda_stream))

    kern_ms: list[float] = []
    value = elapsed_max = 0.0
    clk = None
    if not args.only:
        for _ in range(args.warmup):
            store_step()
        torch.cuda.synchronize(dev)
        probes.zero_()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize(dev)
        with ClockSampler(local) as clk:
            t_all0 = torch.cuda.Event(enable_timing=True)
            t_all1 = torch.cuda.Event(enable_timing=True)
            t_all0.record(stream)
            for k in range(args.steps):
                ev[k][0].record(stream)
                store_step()
                ev[k][1].record(stream)
            t_all1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
        elapsed = t_all0.elapsed_time(t_all1) / 1000.0
        kern_ms = [a.elapsed_time(b) for a, b in ev]
        elapsed_max = max_over_ranks(elapsed)
        value = p.m * args.steps / elapsed_max
        probes_per_edge = int(probes.item()) / (shard * args.steps)
        # spot-check the stored array against the sampled-ID kernel
        if rank == 0:
            ids = np.random.default_rng(1).integers(lo, hi, size=4096, dtype=np.uint64)
            want, _ = pb.edges_at(ids, p, device=dev)
            got = out[torch.from_numpy((ids - np.uint64(lo)).view(np.int64)).to(dev)].cpu().numpy().view(np.uint64)
            assert np.array_equal(got, want), "stored edges disagree with edges_at"
        if args.profile:
            if rank == 0:
                print(json.dumps({"profile": True, "value": value, "kernel_ms": kern_ms}))
            return
    del out
    torch.cuda.empty_cache()

    # ---------------- e2e: reference-facing API, host array out.  Each rank
    # returns E2E_EDGES of its shard as a fresh host array (4 GB; bounded so
    # that 8 ranks do not pin 128 GB of host memory); the edges/s metric is
    # the same.  The native pipeline moves the u32 targets (4 B per edge)
    # over PCIe and fills the (source, target) rows with host threads.
    e2e = None
    if not args.only:
        barrier()
        e2e_n = min(shard, E2E_EDGES)
        e2e_times = []
        # untimed warm-up: at least max(3, W) steps, then until two consecutive
        # steps agree within 10% (at most 10): the first calls pin the host
        # array and wake the host cores and the PCIe link
        e2e_warm_min, e2e_warm = max(3, args.warmup), 0
        prev = None

        def e2e_step() -> float:
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            arr, _ = pb.generate_block(lo, lo + e2e_n, p, device=dev)
            dt = time.perf_counter() - t0
            del arr
            return dt

        while e2e_warm < 10:
            dt = e2e_step()
            e2e_warm += 1
            settled = prev is not None and abs(dt - prev) <= 0.1 * prev
            if ws > 1:  # every rank leaves the warm-up at the same step
                flag = torch.tensor([1 if settled else 0], dtype=torch.int32, device=dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                settled = bool(int(flag.item()))
            prev = dt
            if e2e_warm >= e2e_warm_min and settled:
                break
        for _ in range(args.e2e_steps):
            e2e_times.append(e2e_step())
        e2e_s = max_over_ranks(statistics.median(e2e_times))
        e2e = {"value": e2e_n * ws / e2e_s, "unit": "edges/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": e2e_n * 4 * ws, "edges_per_step_per_gpu": e2e_n,
               "step_seconds_rank0": [round(x, 5) for x in e2e_times], "statistic": "median of the steps", "warmup_steps": e2e_warm,
               "host_threads_per_gpu": int(os.environ["PARBA_HOST_THREADS"]),
               "api": "paper_1602_07106_b200.generate_block(lo, hi, p) -> fresh host (hi-lo,2) uint64 array: "
                      "device generates u32 targets, 4 B/edge over PCIe into pinned staging, host threads "
                      "fill (source, target) rows (C ABI parba_generate_host)",
               "h2d_note": "the generator has no input data: only (n, d, seed, range) scalars cross by value"}

    # ---------------- streaming modes: C3 window, C4 full histogram, C5 the
    # paper's demo (1e12 edges).  Device time per step includes the NCCL
    # reduce of the histogram (N > 1); max over ranks.
    extra = {}
    int_peak = peaks.get("int32_lane_ops_per_s")
    mode_traffic = {}
    mpath = os.path.join(ROOT, "profiles", "r02_mode_traffic.json")
    if os.path.exists(mpath):
        with open(mpath) as fh:
            mode_traffic = json.load(fh)
    if not args.no_extra_modes:
        todo = [("window_c3", C3, C3["K"], 2), ("full_c4", C4, C4["n"], 5), ("window_c5", C5, C5["K"], 1)]
        if args.only:
            todo = [t for t in todo if t[0] == args.only]
        with ClockSampler(local) as clk_modes:
            for name, cfg, K, steps in todo:
                q = pb.GenParams(n=cfg["n"], d=cfg["d"])
                a, b = pb.parallel.shard_range(0, q.m, rank, ws)
                full = name == "full_c4"
                counts = torch.zeros(K, dtype=torch.int32 if full else torch.int64, device=dev)
                prb = torch.zeros(1, dtype=torch.int64, device=dev)
                # warm-up on a slice (attributes, tables, allocator)
                w = min(b - a, 10**9 if not full else b - a)
                pb.parallel.count_shard_device(q, K, b - w, b, counts=counts, probes=prb, device=dev)
                torch.cuda.synchronize(dev)
                balance = None
                if ws > 1:
                    # counting modes: the per-edge cost varies along the ID
                    # space (window hits are denser at low IDs; C4's upper
                    # targets spread over more buckets), so one measured step
                    # on equal shards re-cuts the range into equal-cost
                    # contiguous shards (parallel.balanced_cuts); the counts
                    # do not depend on the cuts
                    cuts0 = [pb.parallel.shard_range(0, q.m, r, ws)[0] for r in range(ws)] + [q.m]
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    pb.parallel.count_shard_device(q, K, a, b, counts=counts, probes=prb, device=dev)
                    e1.record(stream)
                    torch.cuda.synchronize(dev)
                    t_eq = gather(e0.elapsed_time(e1))
                    cuts = pb.parallel.balanced_cuts(cuts0, t_eq)
                    a, b = cuts[rank], cuts[rank + 1]
                    balance = {"partition": "contiguous shards cut to equal cost from one measured step on equal "
                                            "shards (parallel.balanced_cuts)",
                               "equal_shard_ms": t_eq, "cuts": cuts}
                counts.zero_()
                prb.zero_()
                # full histogram on N > 1 GPUs: the reduce fused into the count
                # kernels (every rank adds into the owners' slices over peer
                # memory, parallel.RoutedCounts) when the GPUs can map each
                # other; else count locally + one NCCL reduce of the u32 words
                routed = None
                if full and ws > 1 and os.environ.get("PARBA_ROUTED", "1") != "0":
                    ok = torch.tensor([1 if pb.parallel.routed_ok(q, a, b, dev) else 0], dtype=torch.int32, device=dev)
                    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                    if int(ok.item()):
                        routed = pb.parallel.RoutedCounts.try_create(q, device=dev)
                    if routed is not None:
                        routed.run(a, b)  # warm-up of the routed kernels and the peer mappings
                        # the slices must hold every endpoint before the path is timed
                        tot = (routed.own[: routed.count].to(torch.int64) & 0xFFFFFFFF).sum().reshape(1)
                        dist.all_reduce(tot)
                        if int(tot.item()) != 2 * q.m:  # (the same on every rank) count locally + reduce instead
                            routed.close()
                            routed = None
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(steps):
                    if routed is not None:
                        routed.run(a, b, probes=prb)  # zero, barrier, count into the owners, drain + barrier
                        continue
                    counts.zero_()
                    pb.parallel.count_shard_device(q, K, a, b, counts=counts, probes=prb, device=dev)
                    pb.parallel.reduce_counts(counts, op="reduce")  # u32 words for the full histogram
                e1.record(stream)
                torch.cuda.synchronize(dev)
                t_rank = e0.elapsed_time(e1) / 1000.0
                t = max_over_ranks(t_rank)
                if routed is not None:
                    tot = (routed.own[: routed.count].to(torch.int64) & 0xFFFFFFFF).sum().reshape(1)
                    dist.all_reduce(tot)
                    assert int(tot.item()) == 2 * q.m
                    routed.close()
                else:
                    c64 = pb.parallel.widen_counts(torch, counts, K)
                    if full and rank == 0:
                        assert int(c64.sum().item()) == 2 * q.m
                eps = q.m * steps / t
                ppe = int(prb.item()) / ((b - a) * steps)
                extra[name] = {"edges_per_s": eps, "ms_per_step": 1000 * t / steps,
                               "per_rank_ms_per_step": [1000 * x / steps for x in gather(t_rank)],
                               "n": cfg["n"], "d": cfg["d"], "K": K, "m": q.m, "probes_per_edge": ppe,
                               "steps": steps}
                if balance:
                    extra[name]["balance"] = balance
                if int_peak:
                    ach = eps / ws * 2 * INT_OPS_PER_PROBE  # per GPU, SURVEY 8d convention: 64 lane-ops/edge
                    tb = mode_traffic.get("full_c4_first_batch" if full else "window_c5", {}).get("dram_bytes_per_edge")
                    extra[name]["roofline"] = {
                        "bound": "int", "achieved": ach, "peak": int_peak, "unit": "int32 lane-ops/s per GPU",
                        "frac": ach / int_peak,
                        "traffic": tb * (b - a) if tb is not None else None,
                        "traffic_note": "DRAM bytes of one step on this rank, scaled from the committed ncu capture "
                                        "(profiles/r02_mode_traffic.json: bytes per edge)",
                        "convention": "32 int32 lane-ops per hash probe, 2 probes per edge (SURVEY 8d)",
                        "peak_source": "measured in this run (parba_peak_int32)"}
                if full:
                    extra[name]["path"] = ("partitioned: targets pass with per-CTA bucket histogram, bucket "
                                           "sort in shared memory, shared-memory slice counts (parba_hist.cuh)")
                    if ws > 1:
                        extra[name]["reduce"] = (
                            "fused: count kernels red.add into the owners' slices over peer memory "
                            "(reduce-scatter, parba_degree_full_routed)" if routed is not None
                            else "one reduce of the u32 histogram over the process group")
                del counts
        if extra:
            extra["clocks"] = clk_modes.summary()
    if args.only:
        if rank == 0:
            print(json.dumps({"only": args.only, "modes": extra}), flush=True)
        if ws > 1:
            dist.destroy_process_group()
        return

    kms = gather(statistics.mean(kern_ms))
    if rank != 0:
        dist.destroy_process_group() if ws > 1 else None
        return
    peak, peak_src = _peaks()
    avg_kernel_s = kms[0] / 1000.0
    achieved_gbs = shard * BYTES_PER_EDGE / avg_kernel_s / 1e9
    # DRAM bytes per launch from the committed `ncu --set full` capture of this
    # kernel (profiles/store_traffic.json: dram__bytes_read+write per edge)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "store_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            per_edge = json.load(fh).get("dram_bytes_per_edge")
            traffic = per_edge * shard if per_edge else None
    wo = peaks.get("write_only_gbs")
    line = {
        "metric": METRIC,
        "value": value, "unit": "edges/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * elapsed_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (the generator has no input data)",
        "config": c2_config(ws),
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                     "frac": achieved_gbs / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": shard * BYTES_PER_EDGE,
                     "avg_kernel_ms": kms[0], "per_rank_avg_kernel_ms": kms,
                     # also against the write-only peak measured in this run
                     "write_only_peak_gbs": wo, "frac_of_write_only_peak": achieved_gbs / wo if wo else None},
        "peaks_measured": peaks,
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": args.steps,
        "clocks": clk.summary() if clk else None, "probes_per_edge": probes_per_edge, "modes": extra,
    }
    if args.share_gpu:
        line["debug"] = "share-gpu control-flow check: all ranks on cuda:0 over gloo; not a measurement"
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
