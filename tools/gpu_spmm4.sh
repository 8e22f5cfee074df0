mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spmm_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/tests_spmm_new.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/tests_spmm.log
