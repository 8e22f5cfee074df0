mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
PPCG_GRAM_SBBULK=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_old.json 2> gpurun_out/bench_old.err
