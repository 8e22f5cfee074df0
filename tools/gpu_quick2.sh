# tests + bench (no CPU baseline) + per-kernel breakdown of config 2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2.log 2>&1
