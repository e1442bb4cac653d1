mkdir -p gpurun_out
for f in "c3 1e7" "derby20 1e6" "c2 1e5"; do
  bash tools/ab_n64.sh "A u2 mb6 u2mb5 u2mb6 u4" $f 5 2 >> gpurun_out/ab_i.log 2>&1
done
