mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_k.log 2>&1; echo rc=$? >> gpurun_out/smoke_k.log
BBE_REPORT=gpurun_out/parity_scale_k.json timeout 900 python -m pytest tests/test_gpu_native_scale.py -q -x --timeout 800 > gpurun_out/pytest_scale_k.log 2>&1; echo rc=$? >> gpurun_out/pytest_scale_k.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_c2_k python tools/profile_cfg.py c2 native64 1e5 2 > gpurun_out/ncu_n64_c2_k.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_c2_k 68202000
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_derby20_k python tools/profile_cfg.py derby20 native64 1e6 2 > gpurun_out/ncu_n64_derby20_k.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_derby20_k 2679637000
