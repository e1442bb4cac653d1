#!/bin/bash
# Median NATIVE64 kernel time per library build on one field:  tools/ab_n64.sh "A v1 v2" FIELD SIMS [reps] [rounds]
cd "$(dirname "$0")/.."
F=$2; SIMS=$3; REPS=${4:-5}; ROUNDS=${5:-2}
for r in $(seq 1 "$ROUNDS"); do
  for v in $1; do
    if [ "$v" = A ]; then L=""; else L=paper_2108_02419_b200/_lib/ab/libbbe_$v.so; fi
    BBE_LIB=$L python tools/profile_cfg.py "$F" native64 "$SIMS" "$REPS" 2>&1 | grep -o 'launch [0-9]*: [0-9.]* ms' | tail -n +2 | awk '{print $3}' | sort -n | awk -v v="$v" -v r="$r" -v f="$F" '{a[NR]=$1} END {print f, v, "round", r, "median", a[int((NR+1)/2)], "min", a[1]}'
  done
done
