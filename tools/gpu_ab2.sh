mkdir -p gpurun_out
: > gpurun_out/ab2.txt
timeout 600 python -m pytest tests/test_ozaki_gpu.py -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/ab2.txt
for r in 1 2; do for v in 0 1; do
  echo "== F64COMB=$v rep $r" >> gpurun_out/ab2.txt
  PPCG_OZ_F64COMB=$v timeout 300 python tools/oz_bench.py 2>&1 | grep tsgemm >> gpurun_out/ab2.txt
done; done
for v in 0 1; do
  echo "== warm tts cfg 2 DIGIT_CACHE=$v" >> gpurun_out/ab2.txt
  PPCG_DIGIT_CACHE=$v timeout 600 python tools/tts_warm.py 2 >> gpurun_out/ab2.txt 2>&1
done
