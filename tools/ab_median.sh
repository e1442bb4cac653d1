#!/bin/bash
# Median kernel time of the C2 workload per library build, interleaved over rounds:
#   tools/ab_median.sh "A base v2" [sims] [reps] [rounds]     env BBE_MODE=native|mt
# A = the default in-tree build; other names = paper_2108_02419_b200/_lib/ab/libbbe_NAME.so or
# paper_2108_02419_b200/_lib/ab/NAME/libbbe_sim.so.
SIMS=${2:-100000}; REPS=${3:-20}; ROUNDS=${4:-3}
cd "$(dirname "$0")/.."
for r in $(seq 1 "$ROUNDS"); do
  for v in $1; do
    if [ "$v" = A ]; then L=""; elif [ -f paper_2108_02419_b200/_lib/ab/libbbe_$v.so ]; then L=paper_2108_02419_b200/_lib/ab/libbbe_$v.so; else L=paper_2108_02419_b200/_lib/ab/$v/libbbe_sim.so; fi
    BBE_LIB=$L python tools/profile_c2.py "$SIMS" "$REPS" 2>&1 | grep -o 'launch [0-9]*: [0-9.]* ms' | tail -n +3 | awk -v v="$v" -v r="$r" '{print $3}' | sort -n | awk -v v="$v" -v r="$r" '{a[NR]=$1} END {print v, "round", r, "median", a[int((NR+1)/2)], "min", a[1], "n", NR}'
  done
done
