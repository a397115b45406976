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
