mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native64.py tests/test_gpu_edge.py tests/test_gpu_native_scale.py -q -x --timeout 800 > gpurun_out/pytest_j.log 2>&1; echo rc=$? >> gpurun_out/pytest_j.log
timeout 600 python tools/n64_timing.py --c5 1e8 > gpurun_out/n64_timing_j.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo rc=$? >> gpurun_out/bench_j.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_c5_j python tools/profile_cfg.py c5 native64 1e8 2 > gpurun_out/ncu_n64_c5_j.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_c5_j 267703700000
timeout 600 ncu --set full --import-source on --clock-control none -k regex:exact_kernel -s 1 -c 1 -o gpurun_out/mt_c2_j python tools/profile_mt.py c2 100000 2 > gpurun_out/ncu_mt_c2_j.log 2>&1
bash tools/ncu_export.sh gpurun_out/mt_c2_j 68201961
