"""The C-ABI boundary (CPU): the library builds for sm_100a, loads, and
exports every symbol include/parba_b200.h declares; the product package never
imports the oracle; compute calls fail loudly without a GPU."""

from __future__ import annotations

import ast
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_1602_07106_b200")
HEADER = os.path.join(ROOT, "include", "parba_b200.h")


def _declared_symbols() -> set[str]:
    src = open(HEADER).read()
    return set(re.findall(r"\b(parba_[a-z0-9_]+)\s*\(", src))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1602_07106_b200 import build

    return build.build()


def test_header_declares_the_python_exports():
    from paper_1602_07106_b200 import _lib

    assert _declared_symbols() == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = _declared_symbols() - exported
    assert not missing, missing


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_library_loads_and_answers_without_gpu(lib_path):
    from paper_1602_07106_b200 import _lib

    L = _lib.load(lib_path)
    assert L.parba_version() == 20000
    assert L.parba_device_count() >= 0  # 0 here (no GPU); never fails


def test_abi_validation_errors_without_launch(lib_path):
    # parameter errors are detected on the host side, before any CUDA call
    from paper_1602_07106_b200 import _lib, hashing

    L = _lib.load(lib_path)
    p = hashing.c_params(hashing.HashConfig(), n=10, d=2)
    rc = L.parba_generate(ctypes.byref(p), 5, 3, None, None, None)
    assert rc == _lib.PARBA_EINVAL and b"out of range" in L.parba_last_error()
    bad = hashing.c_params(hashing.HashConfig(), n=10, d=2)
    bad.m = 19
    assert L.parba_generate(ctypes.byref(bad), 0, 1, None, None, None) == _lib.PARBA_EINVAL
    assert b"inconsistent" in L.parba_last_error()
    seedless = hashing.c_params(hashing.HashConfig(), n=10, d=2, n0=3, m0=3)
    assert L.parba_degree_window(ctypes.byref(seedless), 3, 4, 5, None, None, None) == _lib.PARBA_EINVAL


def test_abi_option_flag_and_degree_sequence_validation(lib_path):
    # f3 / f4 parameter errors, all raised before any CUDA call
    from paper_1602_07106_b200 import _lib, hashing

    L = _lib.load(lib_path)
    fake = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    p = hashing.c_params(hashing.HashConfig(), n=10, d=2)
    p.flags = _lib.FLAG_NO_SELF_LOOPS
    assert L.parba_generate(ctypes.byref(p), 0, 2, fake, None, None) == _lib.PARBA_EINVAL
    assert b"require a seed graph" in L.parba_last_error()
    p.flags = 4
    assert L.parba_generate(ctypes.byref(p), 0, 2, fake, None, None) == _lib.PARBA_EINVAL
    assert b"unknown option flags" in L.parba_last_error()
    q = hashing.c_params(hashing.HashConfig(), n=10, d=3, n0=3, m0=3, seed_ptr=512)
    q.flags = _lib.FLAG_NO_PARALLEL_EDGES
    assert L.parba_generate(ctypes.byref(q), 4, q.m, fake, None, None) == _lib.PARBA_EINVAL
    assert b"not a node boundary" in L.parba_last_error()
    assert L.parba_generate(ctypes.byref(q), 3, q.m - 1, fake, None, None) == _lib.PARBA_EINVAL
    assert b"not a node boundary" in L.parba_last_error()
    assert L.parba_edges_at(ctypes.byref(q), fake, 1, fake, None, None) == _lib.PARBA_EINVAL
    assert b"generate_node_edges" in L.parba_last_error()
    r = hashing.c_params(hashing.HashConfig(), n=10, d=2)
    r.degree_prefix = 512
    assert L.parba_generate(ctypes.byref(r), 0, 2, fake, None, None) == _lib.PARBA_EINVAL
    assert b"exactly one of d and degrees" in L.parba_last_error()
    r.d = 0
    assert L.parba_generate(ctypes.byref(r), 0, 2, fake, None, None) == _lib.PARBA_EINVAL
    assert b"rank directory" in L.parba_last_error()
    u = hashing.c_params(hashing.HashConfig(), n=10, d=2)
    assert L.parba_node_of_edges(ctypes.byref(u), fake, 1, fake, 0, None) == _lib.PARBA_EINVAL
    assert b"no prefix index" in L.parba_last_error()
    assert L.parba_node_of_edges(ctypes.byref(u), fake, 1, fake, 7, None) == _lib.PARBA_EINVAL


def test_abi_round2_entry_points_validation(lib_path):
    """The round-2 entry points reject bad input on the host, before CUDA."""
    from paper_1602_07106_b200 import _lib, hashing

    L = _lib.load(lib_path)
    fake = ctypes.c_void_p(256)
    simple = hashing.c_params(hashing.HashConfig(kind=hashing.HashKind.SIMPLE), n=10, d=2)
    assert L.parba_generate_targets(ctypes.byref(simple), 0, 4, fake, None, None) == _lib.PARBA_EINVAL
    assert b"targets-only" in L.parba_last_error()
    crc = hashing.c_params(hashing.HashConfig(), n=10, d=2)
    assert L.parba_generate_targets(ctypes.byref(crc), 3, 1, fake, None, None) == _lib.PARBA_EINVAL
    flagged = hashing.c_params(hashing.HashConfig(), n=10, d=3, n0=3, m0=3, seed_ptr=512)
    flagged.flags = _lib.FLAG_NO_SELF_LOOPS
    assert L.parba_bb_fill(ctypes.byref(flagged), fake, fake, fake, None, None) == _lib.PARBA_EINVAL
    assert b"plain mode only" in L.parba_last_error()
    assert L.parba_debug_mod(99, fake, fake, fake, 1, fake, None) == _lib.PARBA_EINVAL
    assert L.parba_debug_mod_check(0, 1, 10, 0, 5, fake, fake, None) == _lib.PARBA_EINVAL
    devs = np.zeros(2, dtype=np.int32)
    los = np.array([0, 5], dtype=np.uint64)
    his = np.array([5, 21], dtype=np.uint64)  # 21 > m = 20
    assert L.parba_multi_run_shards(ctypes.byref(crc), 2, devs.ctypes.data, los.ctypes.data, his.ctypes.data,
                                    _lib.MULTI_DISCARD, 0, None, None, None) == _lib.PARBA_EINVAL
    assert b"out of range" in L.parba_last_error()
    assert L.parba_multi_run_shards(ctypes.byref(crc), 2, devs.ctypes.data, los.ctypes.data, his.ctypes.data,
                                    9, 0, None, None, None) == _lib.PARBA_EINVAL
    assert L.parba_multi_run_shards(ctypes.byref(crc), 0, None, None, None, _lib.MULTI_DISCARD, 0, None, None,
                                    None) == _lib.PARBA_EINVAL


def test_worker_groups_cover_the_plan():
    """driver.run's split of the reference plan over workers / ranks."""
    import paper_1602_07106_b200 as pb
    from paper_1602_07106_b200 import parallel

    p = pb.GenParams(n=40, d=3, n0=3, seed_edges=np.array([0, 1, 1, 2, 2, 0], dtype=np.uint64))
    plan = pb.plan_batches(p, 10)
    for workers in (1, 2, 3, 5, 12, 20):
        groups = parallel.split_batches(len(plan), workers)
        assert len(groups) == workers and groups[0][0] == 0 and groups[-1][1] == len(plan)
        assert all(a <= b for a, b in groups) and all(groups[k][1] == groups[k + 1][0] for k in range(workers - 1))
        ranges = parallel.group_ranges(p, plan, groups)
        live = [(a, b) for a, b in ranges if b > a]
        assert live[0][0] == p.m0 and live[-1][1] == p.m
        assert all(live[k][1] == live[k + 1][0] for k in range(len(live) - 1))
        assert sum(b - a for a, b in ranges) == p.m - p.m0


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("oracle") or node.level > 0 and node.module == "oracle_compat", f
    for dirpath, _, files in os.walk(os.path.join(PKG, "csrc")):
        for f in files:
            assert "parba_oracle" not in open(os.path.join(dirpath, f)).read(), f


def test_compute_fails_loudly_without_gpu():
    import torch

    import paper_1602_07106_b200 as pb

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = pb.GenParams(n=10, d=2)
    for call in (lambda: pb.generate_block(0, 5, p), lambda: pb.generate_edge(3, p),
                 lambda: pb.degree_counts(p), lambda: pb.h_crc(5, pb.HashConfig()),
                 lambda: pb.resolve_chain_block(np.array([3], dtype=np.uint64), 0, pb.HashConfig())):
        with pytest.raises(pb.GenerationError):
            call()
