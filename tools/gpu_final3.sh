# final state: full GPU suite, smoke, bench, TTS configs 2-4 (cold) + config 2/3 warm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
rm -f gpurun_out/tts_final.jsonl
for c in 3 4; do timeout 1500 python tools/time_to_solution.py $c >> gpurun_out/tts_final.jsonl 2>> gpurun_out/tts_final.err; done
timeout 900 python tools/tts_warm.py 3 > gpurun_out/tts_warm3.json 2>&1
