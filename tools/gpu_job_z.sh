mkdir -p gpurun_out
for f in "c5 1e6" "c1 1e6" "c2 1e5" "derby20 2e5"; do timeout 600 python tools/mt_layout_probe.py $f >> gpurun_out/mt_layout_z.log 2>&1; done
