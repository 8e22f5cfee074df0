# final round evidence: tests, bench (+reference arm), breakdowns, launch list, ncu captures,
# time to solution of configs 1-3 and config-4 iterations
tag=${1:-r1z}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2_$tag.log 2>&1
timeout 600 python tools/iter_breakdown.py 3 3 5 > gpurun_out/breakdown3_$tag.log 2>&1
for c in 1 2 3; do timeout 900 python tools/time_to_solution.py $c >> gpurun_out/tts_$tag.jsonl 2>> gpurun_out/tts_$tag.err; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_$tag.log 2>&1
for w in gram tsgemm; do
  python tools/roofline_capture.py $w > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/roof_${tag}_$w python tools/roofline_capture.py $w > gpurun_out/ncu_roof_$w.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 1 -c 1 \
   -o gpurun_out/prof_${tag}_march python tools/spmm_profile.py 2 march > gpurun_out/ncu_march.log 2>&1
python tools/profile_iter.py 2 2 > gpurun_out/plain.log 2>&1 && for ks in pencil_kernel:1 recombine_kernel:1; do
    k=${ks%%:*}; skip=${ks##*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
        -o gpurun_out/prof_${tag}_$k python tools/profile_iter.py 2 2 > gpurun_out/ncu_${tag}_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_sb_ -s 0 -c 1 \
    -o gpurun_out/prof_${tag}_gram_sb_pair python tools/profile_iter.py 2 3 > gpurun_out/ncu_${tag}_sbtma.log 2>&1
