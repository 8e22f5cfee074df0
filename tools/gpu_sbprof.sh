mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k subblock 2>&1 | tail -2 > gpurun_out/tests_sb.log; timeout 300 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2_sbtma.log 2>&1; python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_sb_tma -s 0 -c 1 \
   -o gpurun_out/prof_sbtma python tools/profile_iter.py 2 3 > gpurun_out/ncu_sbtma.log 2>&1
