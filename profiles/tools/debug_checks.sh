#!/bin/bash
# The GPU test suite against a debug build of the library with device-side bounds checks
# (-DMD_DEBUG_CHECKS: shared-memory list / slab / segment indices, sorted-slot indices; a failed
# check aborts the kernel and the test fails).  compute-sanitizer is not available on the pool.
set -e
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
     --expt-relaxed-constexpr -DMD_DEBUG_CHECKS -o paper_1408_4599_b200/libmardyn_dbg.so \
     paper_1408_4599_b200/csrc/mardyn.cu
MARDYN_LIB=$PWD/paper_1408_4599_b200/libmardyn_dbg.so python -m pytest tests -m gpu -q "$@"
