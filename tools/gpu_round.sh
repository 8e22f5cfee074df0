#!/bin/bash
# One gpurun session: GPU tests, bench line, GEMM microbench, launch list, full ncu of the GEMMs.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
tag=${1:-r1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -30 > gpurun_out/tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_$tag.log 2>&1
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && for k in gram_kernel tsgemm_kernel; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
        -o gpurun_out/prof_${tag}_$k python tools/profile_iter.py 2 2 > gpurun_out/ncu_${tag}_$k.log 2>&1
done
