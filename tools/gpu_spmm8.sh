mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tests.log
SPMM_VARIANTS=2 timeout 900 python tools/spmm_sweep.py 2 3 5 > gpurun_out/spmm_sweep.jsonl 2> gpurun_out/spmm_sweep.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/time_to_solution.py 1 > gpurun_out/tts1.json 2>&1
