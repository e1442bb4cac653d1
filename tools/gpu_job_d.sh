mkdir -p gpurun_out
timeout 300 python tools/profile_cfg.py c1 native 1000 1 > gpurun_out/d_native.log 2>&1; echo rc=$? >> gpurun_out/d_native.log
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python tools/profile_cfg.py c1 native64 1000 1 > gpurun_out/d_n64_memcheck.log 2>&1; echo rc=$? >> gpurun_out/d_n64_memcheck.log
