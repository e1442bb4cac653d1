# round 2: scale parity tests, multi-GPU tally device path, ncu --set full of the C5 NATIVE64 kernel (1e8
# sims: a 1e9 launch is too long for ncu's replay) and of the C2 MT kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edge.py -q -x --timeout 600 -k "multi" > gpurun_out/pytest_multi_g.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi_g.log
BBE_REPORT=gpurun_out/parity_scale_g.json timeout 1500 python -m pytest tests/test_gpu_native_scale.py -q -x --timeout 1400 -s > gpurun_out/pytest_scale_g.log 2>&1; echo rc=$? >> gpurun_out/pytest_scale_g.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_c5_g python tools/profile_cfg.py c5 native64 1e8 2 > gpurun_out/ncu_n64_c5_g.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_c5_g
