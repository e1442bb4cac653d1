mkdir -p gpurun_out
./tools/issue_peak > gpurun_out/issue_peak_b.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_b.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_b.log
for f in c3:1e7 c2:1e5 derby20:1e6 c1:1e6; do
  name=${f%%:*}; n=${f##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_${name}_b python tools/profile_cfg.py $name native64 $n 2 > gpurun_out/ncu_n64_${name}_b.log 2>&1
  bash tools/ncu_export.sh gpurun_out/n64_${name}_b
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native_kernel -s 1 -c 1 -o gpurun_out/n32_c3_b python tools/profile_cfg.py c3 native 1e7 2 > gpurun_out/ncu_n32_c3_b.log 2>&1
bash tools/ncu_export.sh gpurun_out/n32_c3_b
du -sh gpurun_out; ls gpurun_out
