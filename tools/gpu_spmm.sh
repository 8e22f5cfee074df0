mkdir -p gpurun_out
timeout 900 python tools/spmm_sweep.py 2 3 4 5 1 > gpurun_out/spmm_sweep.jsonl 2> gpurun_out/spmm_sweep.err
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/tests_spmm.log
