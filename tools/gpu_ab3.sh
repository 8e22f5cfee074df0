# A/B/C bench of an env toggle: tools/gpu_ab3.sh VAR A B C
var=$1; shift
mkdir -p gpurun_out
for r in 1 2; do for v in "$@"; do
  env $var=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ab_${v}_$r.json 2>> gpurun_out/ab.err
done; done
