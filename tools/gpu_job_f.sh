# round 2: full GPU tests, the new C5 bench (both arms), launch list, ncu --set full of the C5 kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_f.log
timeout 900 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo rc=$? >> gpurun_out/bench_f.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_f.json 2> gpurun_out/bench_ref_f.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 2 --warmup 3 --sweep 0 --cpu-sample 0 --cpu-c-sample 0 --e2e-steps 3 > gpurun_out/ncu_launch_f.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_c5_f python tools/profile_cfg.py c5 native64 1e9 2 > gpurun_out/ncu_n64_c5_f.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_c5_f
nproc > gpurun_out/nproc_f.txt; lscpu | head -20 >> gpurun_out/nproc_f.txt
