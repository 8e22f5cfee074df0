mkdir -p gpurun_out
python tools/profile_iter.py 3 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pencil_kernel -s 0 -c 1 \
  -o gpurun_out/prof_pen192 python tools/profile_iter.py 3 1 > gpurun_out/ncu_pen3.log 2>&1
