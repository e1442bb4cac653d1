mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_c.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_c.log
timeout 600 python tools/n64_timing.py --c5 1e8 > gpurun_out/n64_timing_c.log 2>&1
for f in c3:1e7 derby20:1e6 c2:1e5; do
  name=${f%%:*}; n=${f##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_${name}_c python tools/profile_cfg.py $name native64 $n 2 > gpurun_out/ncu_n64_${name}_c.log 2>&1
  bash tools/ncu_export.sh gpurun_out/n64_${name}_c
done
