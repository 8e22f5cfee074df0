mkdir -p gpurun_out
PPCG_B200_LIB=$PWD/paper_1407_7506_b200/libppcg_b200_prof.so timeout 600 python tools/pencil_phases.py 2 8 > gpurun_out/pencil_phases.txt 2>&1
PPCG_B200_LIB=$PWD/paper_1407_7506_b200/libppcg_b200_prof.so timeout 600 python tools/pencil_phases.py 3 4 > gpurun_out/pencil_phases3.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/tests.log
timeout 600 python tools/pencil_batch_time.py > gpurun_out/pencil_batch.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
