mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for v in "H2_SERIAL=1" "H2_NF_UPW=8"; do
  echo "== $v" >> gpurun_out/ab.log
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/ab.log 2>&1
done
