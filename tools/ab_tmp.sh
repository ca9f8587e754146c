mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s -k "laplace" > gpurun_out/gpu_k.log 2>&1; echo rc=$? >> gpurun_out/gpu_k.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
