#!/bin/bash
# Build the committed (HEAD) sources into paper_1604_01074_b200/libtsmpc_head.so for
# same-box A/B timing against the working tree (TSMPC_LIB=... tools/prof_case.py).
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive HEAD paper_1604_01074_b200/csrc include | tar -x -C "$tmp"
cd "$tmp/paper_1604_01074_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -ldl \
  -o "$root/paper_1604_01074_b200/libtsmpc_head.so" tsmpc_apg.cu tsmpc_sparse.cu tsmpc_sparse_host.cu \
  tsmpc_nccl.cu tsmpc_cache.cu tsmpc_aux.cu tsmpc_capi.cu
rm -rf "$tmp"
