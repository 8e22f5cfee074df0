timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -30 > gpurun_out/tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && for k in gram_kernel tsgemm_kernel; do ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof10_$k python tools/profile_iter.py 2 2 > gpurun_out/ncu10_$k.log 2>&1; done
