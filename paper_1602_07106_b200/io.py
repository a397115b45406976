"""Positional binary edge files fed from the device.

Reference: ``EdgeFileWriter`` / ``_pwrite_all`` (parba/cli.py:109-145): edge i
is stored as two little-endian u64 at byte offset 16*(i - m0), so any range
of edges can be written by any worker in any order and the file is
byte-identical for every schedule.

Uniform-degree families go through the C ABI's ``parba_write_binary``: the
file range is mapped and filled by the host-array pipeline (the device
generates u32 targets, they cross PCIe at 4 B per edge, host threads write
the (source, target) rows straight into the page cache).  Degree sequences
are generated on the GPU in chunks (the store kernel), each chunk copied
into a pinned host buffer while the next one is generated, and a writer
thread ``pwrite``s it at the edge's file offset.
"""

from __future__ import annotations

import os
import queue
import threading

import numpy as np

from . import _lib, driver
from .errors import GenerationError, ParameterError
from .generator import GenParams, _check_block, _cuts, _device

# edges per device chunk (16 B each: 64 MiB chunks, two pinned buffers)
FILE_CHUNK_EDGES = 1 << 22


def _pwrite_all(fd: int, data, offset: int) -> None:
    """pwrite every byte of `data` at `offset` (cli.py:109-118)."""
    view = memoryview(data).cast("B")
    pos = offset
    try:
        while view:
            k = os.pwrite(fd, view, pos)
            pos += k
            view = view[k:]
    except OSError as e:
        raise GenerationError(f"write failed at byte offset {pos}: {e}") from e


class EdgeFileWriter(driver.Consumer):
    """Positional binary writer (cli.py:121-145): edge i lands at byte offset
    16*(i - m0).  ``create=False`` opens an existing file without truncating
    it (other ranks of a multi-process run)."""

    def __init__(self, path: str, m0: int, total_edges: int, create: bool = True):
        if total_edges < 0:
            raise ParameterError(f"total_edges must be >= 0, got {total_edges}")
        self.path = path
        self.m0 = m0
        self.total_edges = total_edges
        flags = os.O_RDWR | os.O_CREAT | (os.O_TRUNC if create else 0)
        self.fd = os.open(path, flags, 0o644)
        if create:
            os.ftruncate(self.fd, 16 * total_edges)

    def new_context(self, worker_id: int) -> int:
        return 0

    def accept_block(self, ctx: int, lo: int, edges: np.ndarray) -> int:
        data = np.ascontiguousarray(edges, dtype="<u8")
        _pwrite_all(self.fd, data, 16 * (lo - self.m0))
        return ctx + data.nbytes

    def merge(self, contexts) -> int:
        return sum(contexts)

    def write_range(self, p: GenParams, lo: int, hi: int, device=None) -> tuple[int, int]:
        """Generate edges lo..hi-1 on the GPU and write them at their file
        offsets.  Returns (bytes written, hash probes).

        Uniform degree: the C ABI's ``parba_write_binary`` maps the file range
        and fills it with the host-array pipeline (u32 targets over PCIe, rows
        written into the page cache by a team of host threads).  Degree
        sequences: device chunks, pinned buffers, one ``pwrite`` thread."""
        _check_block(lo, hi, p)
        if lo == hi:
            return 0, 0
        torch, dev = _device(device)
        L = _lib.load()
        if p.d is not None and os.environ.get("PARBA_WRITER_PWRITE") != "1":
            import ctypes

            if lo < self.m0 or 16 * (hi - self.m0) > os.fstat(self.fd).st_size:
                raise ParameterError(f"edges [{lo}, {hi}) fall outside the file's range")
            cp, _keep = p._host_params()
            probes = ctypes.c_uint64(0)
            idx = dev.index if dev.index is not None else torch.cuda.current_device()
            _lib.check(L.parba_write_binary(ctypes.byref(cp), lo, hi, self.fd, self.m0, ctypes.byref(probes), idx))
            return 16 * (hi - lo), int(probes.value)
        total = hi - lo
        cuts = _cuts(p, lo, hi, min(total, FILE_CHUNK_EDGES))  # node-aligned under option flags
        spans = list(zip(cuts, cuts[1:]))
        chunk = max(b - a for a, b in spans)
        nbuf = 2
        work: queue.Queue = queue.Queue(maxsize=nbuf)
        free: queue.Queue = queue.Queue()
        errors: list[BaseException] = []

        def writer():
            while True:
                item = work.get()
                if item is None:
                    return
                k, a, n, host, ev = item
                try:
                    ev.synchronize()
                    _pwrite_all(self.fd, host[: 2 * n].numpy(), 16 * (a - self.m0))
                except BaseException as e:  # surfaced after the loop
                    errors.append(e)
                free.put(k)

        with torch.cuda.device(dev):
            comp = torch.cuda.current_stream(dev)
            copy = torch.cuda.Stream(dev)
            dbufs = [torch.empty(2 * chunk, dtype=torch.int64, device=dev) for _ in range(nbuf)]
            hbufs = [torch.empty(2 * chunk, dtype=torch.int64, pin_memory=True) for _ in range(nbuf)]
            for k in range(nbuf):
                free.put(k)
            probes = torch.zeros(1, dtype=torch.int64, device=dev)
            cp = p._device_params(dev)
            th = threading.Thread(target=writer, daemon=True)
            th.start()
            try:
                for a, b in spans:
                    n = b - a
                    k = free.get()  # host buffer k (and device buffer k) are free again
                    _lib.check(L.parba_generate(cp, a, a + n, dbufs[k].data_ptr(), probes.data_ptr(),
                                                comp.cuda_stream))
                    made = torch.cuda.Event()
                    made.record(comp)
                    copy.wait_event(made)
                    with torch.cuda.stream(copy):
                        hbufs[k][: 2 * n].copy_(dbufs[k][: 2 * n], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(copy)
                    work.put((k, a, n, hbufs[k], ev))
                    if errors:
                        break
            finally:
                work.put(None)
                th.join()
            if errors:
                raise errors[0]
            return 16 * total, int(probes.item())

    def close(self) -> None:
        os.close(self.fd)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def write_edges_binary(path: str, p: GenParams, device=None) -> tuple[int, int]:
    """Whole-graph binary file (`parba generate -o`, cli.py:279-297): edges
    m0..m-1 at offsets 16*(i - m0).  Returns (bytes, probes)."""
    with EdgeFileWriter(path, p.m0, p.m - p.m0) as w:
        return w.write_range(p, p.m0, p.m, device=device)
