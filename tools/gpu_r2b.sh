# round-2 evidence with the emulated FP64 products: GPU tests, smoke, bench (+reference arm),
# breakdown, launch list, ncu of the emulated kernels
tag=${1:-r2b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 --durations=10 > gpurun_out/tests_$tag.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 python tools/iter_breakdown.py 2 5 10 > gpurun_out/breakdown2_$tag.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_small_$tag.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch_$tag.log 2>&1
python tools/oz_one.py ts && timeout 500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_oz_ts|k_slice_rows" -s 2 -c 2 -o gpurun_out/oz_ts_$tag python tools/oz_one.py ts > gpurun_out/ncu_ts_$tag.log 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gram|k_slice_cols|k_colmax|k_gram_reduce" \
  -s 6 -c 6 -o gpurun_out/oz_gram_$tag python tools/oz_one.py gram > gpurun_out/ncu_gram_$tag.log 2>&1
