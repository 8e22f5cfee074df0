mkdir -p gpurun_out
SPMM_VARIANTS=0,1,2 timeout 900 python tools/spmm_sweep.py 2 3 5 4 1 > gpurun_out/spmm_sweep.jsonl 2> gpurun_out/spmm_sweep.err
timeout 900 python -m pytest tests/test_spmm_gpu.py -q -x 2>&1 | tail -5 > gpurun_out/tests_spmm.log
