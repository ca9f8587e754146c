mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or dense or fly or shard" > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
python tools/mv_probe.py > gpurun_out/mv.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"matvec|up_kernel|coupling|permute|down_kernel" --log-file gpurun_out/mv_launches.csv python tools/mv_probe.py > gpurun_out/ncu_mv.log 2>&1
echo rc=$?
