mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q -s > gpurun_out/gpu_shard.log 2>&1; echo rc=$? >> gpurun_out/gpu_shard.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
