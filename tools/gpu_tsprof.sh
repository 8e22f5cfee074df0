mkdir -p gpurun_out
python tools/roofline_capture.py tsgemm > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_oz_ts \
  -o gpurun_out/roof_r02g_tsgemm python tools/roofline_capture.py tsgemm > gpurun_out/ncu_roof_tsgemm.log 2>&1
timeout 1500 python -m pytest tests/test_solver_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/solver_tests.log
