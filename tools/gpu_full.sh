# full GPU suite, bench (no CPU legs), e2e phases, digit-cache A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
PPCG_DIGIT_CACHE=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_nocache.json 2> gpurun_out/bench_nocache.err
timeout 600 python tools/e2e_phases.py 2 20 5 > gpurun_out/e2e_phases.txt 2>&1
