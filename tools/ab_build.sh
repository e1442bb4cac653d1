#!/bin/bash
# Build variant libraries of the simulator for A/B timing on the GPU box:
#   tools/ab_build.sh NAME "-DFLAG=V ..."   ->  paper_2108_02419_b200/_lib/ab/libbbe_NAME.so
# Run with BBE_LIB=paper_2108_02419_b200/_lib/ab/libbbe_NAME.so python tools/profile_c2.py
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2108_02419_b200/_lib/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr $2 -o "paper_2108_02419_b200/_lib/ab/libbbe_$1.so" \
    paper_2108_02419_b200/csrc/bbe_sim.cu paper_2108_02419_b200/csrc/host_mt.cpp -ldl
echo "built paper_2108_02419_b200/_lib/ab/libbbe_$1.so"
