mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spmm_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/tests.log
SPMM_VARIANTS=0,1,2 timeout 900 python tools/spmm_sweep.py 2 3 5 4 1 > gpurun_out/spmm_sweep.jsonl 2> gpurun_out/spmm_sweep.err
python tools/spmm_profile.py 2 march > gpurun_out/spmm_prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 1 -c 1 \
   -o gpurun_out/prof_r1k_march python tools/spmm_profile.py 2 march > gpurun_out/ncu_march.log 2>&1
