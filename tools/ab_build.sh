#!/bin/bash
# Build variant libraries of the simulator for A/B timing on the GPU box:
#   tools/ab_build.sh NAME "-DFLAG=V ..."   ->  paper_2108_02419_b200/_lib/ab/libbbe_NAME.so
# Run with BBE_LIB=paper_2108_02419_b200/_lib/ab/libbbe_NAME.so python tools/profile_c2.py
set -e
cd "$(dirname "$0")/.."
OUT=paper_2108_02419_b200/_lib/ab/$1
mkdir -p "$OUT"
make -s -j8 LIBDIR="$OUT" NVEXTRA="$2" "$OUT/libbbe_sim.so"
cp "$OUT/libbbe_sim.so" "paper_2108_02419_b200/_lib/ab/libbbe_$1.so"
rm -f "$OUT/libbbe_sim.so"  # one copy per variant travels to the GPU box (.gpurunignore drops $OUT)
echo "built paper_2108_02419_b200/_lib/ab/libbbe_$1.so"
