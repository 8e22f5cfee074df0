mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/tests.log
timeout 1500 python tools/iter_breakdown.py 5 2 3 64 1024 > gpurun_out/breakdown5s_c.log 2>&1
