mkdir -p gpurun_out
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_bulk_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_sb96 python tools/profile_iter.py 2 2 > gpurun_out/ncu_sb.log 2>&1
