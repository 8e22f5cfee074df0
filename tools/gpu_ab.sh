# tests + A/B bench of an env toggle: tools/gpu_ab.sh VAR VAL_A VAL_B
var=$1; a=$2; b=$3
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tests.log
for r in 1 2; do for v in $a $b; do
  env $var=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ab_${v}_$r.json 2>> gpurun_out/ab.err
done; done
