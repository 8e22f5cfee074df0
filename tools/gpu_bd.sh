mkdir -p gpurun_out
timeout 600 python tools/iter_breakdown.py 2 120 10 > gpurun_out/breakdown2_locked.log 2>&1
timeout 600 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2.log 2>&1
timeout 900 python tools/iter_breakdown.py 3 5 5 > gpurun_out/breakdown3.log 2>&1
