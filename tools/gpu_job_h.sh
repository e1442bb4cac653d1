# unit53 draws: NATIVE64 parity (bit-exact vs the oracle), timing, ncu of the C5 kernel, short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native64.py tests/test_gpu_edge.py -q -x --timeout 600 > gpurun_out/pytest_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_h.log
timeout 600 python tools/n64_timing.py --c5 1e8 > gpurun_out/n64_timing_h.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_c5_h python tools/profile_cfg.py c5 native64 1e8 2 > gpurun_out/ncu_n64_c5_h.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_c5_h
