mkdir -p gpurun_out
SPMM_VARIANTS=2 timeout 900 python tools/spmm_sweep.py 2 > gpurun_out/spmm_sweep.jsonl 2> gpurun_out/spmm_sweep.err
timeout 300 python tools/time_to_solution.py 1 > gpurun_out/tts1.json 2>&1
PPCG_PENCIL_EIG=jacobi timeout 300 python tools/time_to_solution.py 1 > gpurun_out/tts1_jac.json 2>&1
timeout 300 python tools/iter_breakdown.py 1 20 20 > gpurun_out/breakdown1.log 2>&1
PPCG_PENCIL_EIG=jacobi timeout 300 python tools/iter_breakdown.py 1 20 20 > gpurun_out/breakdown1_jac.log 2>&1
