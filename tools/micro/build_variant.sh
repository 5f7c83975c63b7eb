#!/bin/bash
# dev helper (not product): build libheap_<name>.so with extra -D flags for A/B engine probes
# usage: tools/micro/build_variant.sh NAME [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/../.."
NAME=$1; shift
INC=$(python -c "from paper_2405_07079_b200 import _native as n; print(n.nccl_dirs()[0])")
LIBD=$(python -c "from paper_2405_07079_b200 import _native as n; print(n.nccl_dirs()[1])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" -I "$INC" \
  -o paper_2405_07079_b200/libheap_$NAME.so paper_2405_07079_b200/csrc/heap.cu -L "$LIBD" -l:libnccl.so.2 -Xlinker -rpath,"$LIBD"
