mkdir -p gpurun_out
timeout 1500 python tools/iter_breakdown.py 5 2 3 64 1024 > gpurun_out/breakdown5s_r02g.log 2>&1
