#!/bin/bash
# Time the C2 native workload for the default build (A) and A/B variants: tools/ab_run.sh "A F G" [sims]
SIMS=${2:-100000}
for v in $1; do
  if [ "$v" = A ]; then L=""; else L=paper_2108_02419_b200/_lib/ab/libbbe_$v.so; fi
  BBE_LIB=$L python tools/profile_c2.py $SIMS 6 2>&1 | tail -2 | sed "s/^/$v($SIMS): /"
done
