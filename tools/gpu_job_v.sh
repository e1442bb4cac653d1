mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native_kernel -s 1 -c 1 -o gpurun_out/n32_derby20_v python tools/profile_cfg.py derby20 native 1e6 2 > gpurun_out/ncu_n32_derby20_v.log 2>&1
bash tools/ncu_export.sh gpurun_out/n32_derby20_v 2679637000
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_derby20_v python tools/profile_cfg.py derby20 native64 1e6 2 > gpurun_out/ncu_n64_derby20_v.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_derby20_v 2679637000
