mkdir -p gpurun_out
rm -f gpurun_out/ab.log
for v in "H2_NF_UPW=8" "H2_NF_THREADS=128" "H2_NF_THREADS=128 H2_NF_UPW=4" "H2_NF_THREADS=128 H2_NF_UPW=16" "H2_SERIAL=1 H2_NF_THREADS=128"; do
  echo "== $v" >> gpurun_out/ab.log
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/ab.log 2>&1
done
