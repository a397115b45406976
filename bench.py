#!/usr/bin/env python
"""Benchmark: edges generated / s (device-timed) for the Sanders-Schulz BA
generator on B200 -- BASELINE.json's metric on its configs[1] (store mode,
n=1e8, d=10, m=1e9 int64 pairs written to HBM), the fixed graph's edge-ID
range sharded over the GPUs as configs[1] prescribes (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One JSON line on rank 0.  `value` = whole-job edges/s with the output
resident in HBM; `e2e` = the same metric through the reference-facing API
`generate_block(lo, hi, p)` returning a host array (device->host copy inside
the timed region); `roofline` = the store kernel's algorithmic 16 B/edge
write rate against the measured HBM peak; `cpu_baseline` = the CPU oracle
port (reference algorithm in C) on a bounded sample, all host cores.
`--impl reference` times that CPU implementation alone.
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
METRIC = "edges generated/sec (device-timed) at 1/2/4/8 B200; % of HBM/int roofline"  # BASELINE.json metric
BYTES_PER_EDGE = 16               # algorithmic HBM bytes per stored edge
E2E_EDGES = 250_000_000  # edges per GPU returned to the host per e2e step (4 GB)
WRITE_ONLY_GBS = 6867.6  # write-only HBM peak measured by tools/micro.cu on a B200 of this pool
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


def c2_config(ws: int) -> dict:
    """The workload both arms report (BASELINE.json configs[1])."""
    m = C2["n"] * C2["d"]
    return {"workload": "configs[1]: store mode, n=1e8, d=10, m=1e9 edges -> (m,2) u64 pairs (16 GB) "
                        "in HBM, contiguous edge-ID shards over the GPUs (total work fixed)",
            "n": C2["n"], "d": C2["d"], "m": m, "shard_edges": m // ws,
            "parallelism": f"edge-range shards x{ws} (no collective in store mode)",
            "l2": "output 16 GB/N >> 126 MB L2: no flush needed between steps"}


def run_reference(args) -> None:
    rank, ws, _ = _dist()
    if rank != 0:
        return
    samples = []
    n_edges = None
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(sample_edges=n_edges, budget_s=4.0)
        n_edges = n_edges or cb["sample_edges"]
        if k >= args.warmup:
            samples.append(cb)
    value = statistics.median(s["value"] for s in samples)
    line = {"impl": "reference", "metric": METRIC,
            "value": value, "unit": "edges/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * n_edges / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": c2_config(ws) | {"sample_edges": n_edges,
                                       "reference_step": "a bounded CPU sample of the workload per step"},
            "cpu_baseline": {k: samples[-1][k] for k in ("kind", "cores", "sample")} | {"value": value, "unit": "edges/s"},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-modes", action="store_true")
    ap.add_argument("--profile", action="store_true", help="store kernel only (for ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile else args.warmup

    if args.impl == "reference":
        run_reference(args)
        return

    rank, ws, local = _dist()
    # CPU baseline first: the oracle is plain C, but keep it out of the
    # timed GPU region and before CUDA work on rank 0 (N=1 only).
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile:
        cpu = cpu_baseline()

    import torch
    import torch.distributed as dist

    import paper_1602_07106_b200 as pb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    L = pb._lib.load()

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- store mode, C2 (headline): BASELINE.json configs[1] is
    # one fixed graph (n=1e8, d=10) "sharded by contiguous edge-ID ranges over
    # 1/2/4/8 GPUs", so total work is fixed as N grows (strong scaling).
    p = pb.GenParams(**C2)
    lo, hi = pb.parallel.shard_range(0, p.m, rank, ws)
    shard = hi - lo
    out = torch.empty((shard, 2), dtype=torch.int64, device=dev)
    probes = torch.zeros(1, dtype=torch.int64, device=dev)
    cp = p._device_params(dev)
    stream = torch.cuda.current_stream(dev)

    def store_step():
        pb._lib.check(L.parba_generate(cp, lo, hi, out.data_ptr(), probes.data_ptr(), stream.cuda_stream))

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
    peak, peak_src = _peaks()
    avg_kernel_s = statistics.mean(kern_ms) / 1000.0
    achieved_gbs = shard * BYTES_PER_EDGE / avg_kernel_s / 1e9
    # spot-check the stored array against the sampled-ID kernel (no oracle on this path)
    if rank == 0:
        import numpy as np

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
    # the same.
    barrier()
    e2e_n = min(shard, E2E_EDGES)
    e2e_times = []
    for k in range(1 + args.e2e_steps):
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        arr, _ = pb.generate_block(lo, lo + e2e_n, p, device=dev)
        dt = time.perf_counter() - t0
        if k:
            e2e_times.append(dt)
        del arr
    e2e_s = max_over_ranks(statistics.median(e2e_times))
    e2e = {"value": e2e_n * ws / e2e_s, "unit": "edges/s", "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": e2e_n * 16, "edges_per_step_per_gpu": e2e_n,
           "api": "paper_1602_07106_b200.generate_block(lo, hi, p) -> host (hi-lo,2) uint64 (pinned), "
           "chunked device generation overlapped with D2H",
           "h2d_note": "the generator has no input data: only (n, d, seed, range) scalars cross by value"}

    # ---------------- extra modes: C3 streaming window, C4 full histogram
    extra = {}
    if not args.no_extra_modes:
        for name, cfg, K in (("window_c3", C3, C3["K"]), ("full_c4", C4, C4["n"])):
            q = pb.GenParams(n=cfg["n"], d=cfg["d"])
            a, b = pb.parallel.shard_range(0, q.m, rank, ws)
            counts = torch.zeros(K, dtype=torch.int32 if name == "full_c4" else torch.int64, device=dev)
            prb = torch.zeros(1, dtype=torch.int64, device=dev)
            steps = 2 if name == "window_c3" else 5
            pb.parallel.count_shard_device(q, K, a, b, counts=counts, probes=prb, device=dev)
            torch.cuda.synchronize(dev)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                counts.zero_()
                pb.parallel.count_shard_device(q, K, a, b, counts=counts, probes=prb, device=dev)
                pb.parallel.reduce_counts(counts, op="reduce")  # u32 words for the full histogram
            e1.record(stream)
            torch.cuda.synchronize(dev)
            c64 = pb.parallel.widen_counts(torch, counts, K)  # C4's counts are u32 in HBM; widened for the check
            t = max_over_ranks(e0.elapsed_time(e1) / 1000.0)
            if name == "full_c4" and rank == 0:
                assert int(c64.sum().item()) == 2 * q.m
            extra[name] = {"edges_per_s": q.m * steps / t, "ms_per_step": 1000 * t / steps,
                           "n": cfg["n"], "d": cfg["d"], "K": K, "m": q.m,
                           "int_ops_per_s_convention": q.m * steps / t * 2 * INT_OPS_PER_PROBE}
            if name == "full_c4":
                extra[name]["path"] = ("partitioned: targets pass with per-CTA bucket histogram, bucket "
                                       "sort in shared memory, shared-memory slice counts (parba_hist.cuh); "
                                       "no per-edge global atomics")
            del counts

    if rank != 0:
        dist.destroy_process_group() if ws > 1 else None
        return
    # DRAM bytes per launch from the committed `ncu --set full` capture of this
    # kernel (profiles/store_traffic.json: dram__bytes_read+write per edge)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "store_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            per_edge = json.load(fh).get("dram_bytes_per_edge")
            traffic = per_edge * shard if per_edge else None
    line = {
        "metric": METRIC,
        "value": value, "unit": "edges/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * elapsed_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (the generator has no input data)",
        "config": c2_config(ws),
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                     "frac": achieved_gbs / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": shard * BYTES_PER_EDGE,
                     # also against a write-only peak measured on this pool
                     # (tools/micro.cu, profiles/r01_micro.json: 6867.6 GB/s)
                     "frac_of_write_only_peak": achieved_gbs / WRITE_ONLY_GBS,
                     "avg_kernel_ms": statistics.mean(kern_ms)},
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": args.steps,
        "clocks": clk.summary(), "probes_per_edge": probes_per_edge, "modes": extra,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
