mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_native64.py -q -x --timeout 600 > gpurun_out/pytest_p.log 2>&1; echo rc=$? >> gpurun_out/pytest_p.log
for f in "c3 1e7" "c1 1e6" "c2 1e5" "derby20 1e6"; do
  bash tools/ab_n64.sh "A u53alu" $f 7 3 >> gpurun_out/ab_p.log 2>&1
done
