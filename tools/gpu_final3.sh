mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
timeout 600 python tools/e2e_phases.py 2 20 8 > gpurun_out/e2e_phases.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
