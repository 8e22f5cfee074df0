mkdir -p gpurun_out
: > gpurun_out/ab4.txt
for r in 1 2; do for v in 32 64; do
  echo "== TBN=$v EPI=8 rep $r" >> gpurun_out/ab4.txt
  PPCG_OZ_EPI=8 PPCG_OZ_TBN=$v timeout 300 python tools/oz_bench.py 2>&1 | grep tsgemm >> gpurun_out/ab4.txt
done; done
