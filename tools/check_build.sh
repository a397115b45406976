#!/usr/bin/env bash
# Build the library with device-side invariant checks (queue ring never
# overflows, stage cells in range, node-kernel writes in range: a violated
# check traps) and run the GPU parity suite against it.  On the GPU box:
#   bash tools/check_build.sh
set -eu
mkdir -p build_ab
python -c "from paper_1602_07106_b200 import build; build.build(out='build_ab/lib_checks.so', defines={'PARBA_DEBUG_CHECKS': 1})"
PARBA_LIB=build_ab/lib_checks.so python -m pytest tests -m gpu -q -x
