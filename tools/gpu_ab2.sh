mkdir -p gpurun_out
: > gpurun_out/ab5.txt
for v in 5 2 3 4; do
  echo "== PPCG_RECOMB_MINB64=$v" >> gpurun_out/ab5.txt
  PPCG_RECOMB_MINB64=$v timeout 600 python tools/iter_breakdown.py 3 3 4 2>&1 | grep -E "cfg 3|recombine" >> gpurun_out/ab5.txt
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "recomb or subblock or update" 2>&1 | tail -2 >> gpurun_out/ab5.txt
