# round-end evidence: tests, smoke, bench (+reference arm), breakdowns, launch list, ncu captures
tag=${1:-r02g}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2_$tag.log 2>&1
timeout 300 python tools/iter_breakdown.py 2 120 10 > gpurun_out/breakdown2_locked_$tag.log 2>&1
timeout 600 python tools/iter_breakdown.py 3 3 5 > gpurun_out/breakdown3_$tag.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_$tag.log 2>&1
for w in gram tsgemm; do
  python tools/roofline_capture.py $w > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/roof_${tag}_$w python tools/roofline_capture.py $w > gpurun_out/ncu_roof_$w.log 2>&1
done
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && for ks in pencil_kernel:1 recombine_kernel:1 spmm_stencil:1 gram_sb_:1; do
    k=${ks%%:*}; skip=${ks##*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
        -o gpurun_out/prof_${tag}_$k python tools/profile_iter.py 2 3 > gpurun_out/ncu_${tag}_$k.log 2>&1
done
