mkdir -p gpurun_out
for w in 12 16; do PPCG_GRAM_MINWAVES=$w timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; done
