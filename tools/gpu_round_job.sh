# One GPU call: full GPU tests, smoke, bench + reference arm, ncu launch list, full captures (native, MT).
# usage (on the box): bash tools/gpu_round_job.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --sweep 0 --cpu-sample 0 --cpu-c-sample 0 > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:native_kernel -s 2 -c 1 -o gpurun_out/native_$TAG python tools/profile_c2.py 100000 4 > gpurun_out/ncu_nat_$TAG.log 2>&1
BBE_MODE=mt ncu --set full --import-source on --clock-control none -k regex:exact_kernel -s 1 -c 1 -o gpurun_out/mt_$TAG python tools/profile_c2.py 100000 3 > gpurun_out/ncu_mt_$TAG.log 2>&1
ls gpurun_out
