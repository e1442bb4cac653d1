mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_native64.py tests/test_gpu_native.py -q -x --timeout 600 > gpurun_out/pytest_gpu_e.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_e.log
timeout 600 python tools/n64_timing.py --c5 1e8 > gpurun_out/n64_timing_e.log 2>&1
