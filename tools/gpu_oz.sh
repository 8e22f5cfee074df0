# emulation tests, A/B timing of the products, bench without the CPU legs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ozaki_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/oz_tests.log
timeout 300 python tools/oz_bench.py > gpurun_out/oz_ab.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
