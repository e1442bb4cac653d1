mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mt.py tests/test_gpu_inject.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py tests/test_gpu_acceptance.py tests/test_session_exchange.py tests/test_gpu_session.py -q -x --timeout 900 > gpurun_out/pytest_l.log 2>&1; echo rc=$? >> gpurun_out/pytest_l.log
BBE_MODE=mt bash tools/ab_median.sh "mtbase mtkey mtkey_mb4" 100000 12 3 > gpurun_out/ab_mt_l.log 2>&1
