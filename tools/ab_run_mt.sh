#!/bin/bash
# MT-mode A/B: tools/ab_run_mt.sh "A M5 M6"
for v in $1; do
  if [ "$v" = A ]; then L=""; else L=paper_2108_02419_b200/_lib/ab/libbbe_$v.so; fi
  BBE_MODE=mt BBE_LIB=$L python tools/profile_c2.py 100000 4 2>&1 | tail -2 | sed "s/^/$v: /"
done
