#!/bin/bash
# Per-function stack / spill report of tsmpc_sparse.cu (ptxas -v), demangled names.
# usage: tools/ptxas_spills.sh [source.cu]  (default: the working tree's tsmpc_sparse.cu)
SRC=${1:-paper_1604_01074_b200/csrc/tsmpc_sparse.cu}
INC=$(cd "$(dirname "$0")/.." && pwd)/paper_1604_01074_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I"$INC" -Xptxas -v -c -o /tmp/ptxas_spills.o "$SRC" 2>&1 |
  awk '/Function properties for|Compiling entry function/ {name=$NF} /spill/ {print name": "$0}' |
  sed "s/'//g" | c++filt | sed 's/(tsmpc::LaunchWin)//' | awk '$0 !~ /0 bytes spill stores, 0 bytes spill loads/'
