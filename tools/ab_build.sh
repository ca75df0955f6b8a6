#!/bin/bash
# Build an alternative libmdhp.so from a given eval.cuh variant into tools/ab/<name>/ for A/B runs
# (MDHP_LIB=tools/ab/<name>/libmdhp.so python bench.py ...).  Usage: tools/ab_build.sh name eval.cuh
set -e
name=$1; ev=$2
d=/root/repo/tools/ab/$name; mkdir -p $d/csrc
cp /root/repo/paper_2411_10258_b200/csrc/*.cu /root/repo/paper_2411_10258_b200/csrc/*.cuh $d/csrc/
cp $ev $d/csrc/eval.cuh
cd $d/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I/root/repo/paper_2411_10258_b200/csrc -o $d/libmdhp.so abi.cu pack.cu fit.cu exact.cu seq.cu dense.cu features.cu
echo built $d/libmdhp.so
