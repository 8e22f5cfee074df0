#!/bin/bash
# One gpurun session: GPU tests, bench line (+ CPU baseline), GEMM microbench, per-call and
# per-kernel iteration breakdowns, the bench's ncu launch list, and full ncu captures of the
# top kernels (each only after the same command exited 0 without ncu).
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_round.sh r1d'
tag=${1:-r1}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -30 > gpurun_out/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep.json 2>&1
timeout 300 python tools/call_timing.py 2 5 5 > gpurun_out/calls2_$tag.log 2>&1
timeout 300 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2_$tag.log 2>&1
timeout 600 python tools/iter_breakdown.py 3 3 5 > gpurun_out/breakdown3_$tag.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_$tag.log 2>&1
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && for ks in gram_kernel:3 tsgemm_kernel:3 pencil_kernel:1 recombine_kernel:1 spmm_csr:2; do
    k=${ks%%:*}; skip=${ks##*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
        -o gpurun_out/prof_${tag}_$k python tools/profile_iter.py 2 2 > gpurun_out/ncu_${tag}_$k.log 2>&1
done
