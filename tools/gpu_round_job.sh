# One GPU call: full GPU tests, smoke, bench + reference arm, ncu launch list, full captures of the
# NATIVE64 C5 kernel (1e8 races: a 1e9 launch is too long for ncu's replay) and the MT C2 kernel.
# usage (on the box): bash tools/gpu_round_job.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 1200 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --sweep 0 --cpu-sample 0 --cpu-c-sample 0 --e2e-steps 3 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:native64_kernel -s 1 -c 1 -o gpurun_out/n64_c5_$TAG python tools/profile_cfg.py c5 native64 1e8 2 > gpurun_out/ncu_n64_c5_$TAG.log 2>&1
bash tools/ncu_export.sh gpurun_out/n64_c5_$TAG 267703700000
timeout 600 ncu --set full --import-source on --clock-control none -k regex:exact_kernel -s 1 -c 1 -o gpurun_out/mt_c2_$TAG python tools/profile_mt.py c2 100000 2 > gpurun_out/ncu_mt_c2_$TAG.log 2>&1
bash tools/ncu_export.sh gpurun_out/mt_c2_$TAG 68201961
ls gpurun_out
