# same-box A/B of two library builds: tools/gpu_ab_lib.sh <script and args...>
mkdir -p gpurun_out
: > gpurun_out/ab_lib.txt
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export PPCG_B200_LIB=$PWD/paper_1407_7506_b200/libppcg_b200_old.so; else unset PPCG_B200_LIB; fi
  echo "== $v $r" >> gpurun_out/ab_lib.txt
  timeout 600 python "$@" >> gpurun_out/ab_lib.txt 2>&1
done; done
