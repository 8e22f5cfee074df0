mkdir -p gpurun_out
python tools/spmm_profile.py 2 march > gpurun_out/spmm_prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm -s 2 -c 2 \
   -o gpurun_out/prof_spmm_march python tools/spmm_profile.py 2 march > gpurun_out/ncu_spmm.log 2>&1
