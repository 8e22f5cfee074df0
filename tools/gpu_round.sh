set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_solver_gpu.py -m gpu -q --timeout 300 2>&1 | tail -5 > gpurun_out/t3.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && for k in pencil_kernel recombine_kernel gram_kernel; do ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof2_$k python tools/profile_iter.py 2 2 > gpurun_out/ncu2_$k.log 2>&1; done
