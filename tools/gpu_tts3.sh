# time to solution configs 1-4 (emulated products, digit cache on), config 2/3 with the cache off
mkdir -p gpurun_out
rm -f gpurun_out/tts_r02g.jsonl gpurun_out/tts_r02g_nocache.jsonl
for c in 1 2 3 4; do timeout 1500 python tools/time_to_solution.py $c >> gpurun_out/tts_r02g.jsonl 2>> gpurun_out/tts_r02g.err; done
for c in 2 3; do PPCG_DIGIT_CACHE=0 timeout 1200 python tools/time_to_solution.py $c >> gpurun_out/tts_r02g_nocache.jsonl 2>> gpurun_out/tts_r02g.err; done
