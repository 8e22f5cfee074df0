mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_solver_gpu.py tests/test_golden_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x 2>&1 | tail -6 > gpurun_out/ptd_tests.log
timeout 600 python tools/pencil_batch_time.py > gpurun_out/pencil_batch.txt 2>&1
