#!/bin/bash
# Build an alternative libmdhp.so of the current sources with extra nvcc flags into
# tools/ab/<name>/ for A/B runs (MDHP_LIB=tools/ab/<name>/libmdhp.so ...).
# Usage: tools/ab_build_flags.sh name "-DFOO=1 ..."
set -e
name=$1; flags=$2
d=/root/repo/tools/ab/$name; mkdir -p $d
cd /root/repo/paper_2411_10258_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared $flags -o $d/libmdhp.so abi.cu pack.cu fit.cu exact.cu seq.cu dense.cu features.cu
echo built $d/libmdhp.so
