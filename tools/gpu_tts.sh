# time to solution (public ppcg_solve) for BASELINE configs 1-4, emulated FP64 products (default)
# and the DMMA kernels (PPCG_FP64_EMU=0) for configs 2-3
mkdir -p gpurun_out
for c in 1 2 3 4; do timeout 1200 python tools/time_to_solution.py $c >> gpurun_out/tts_r02.jsonl 2>> gpurun_out/tts_r02.err; done
for c in 2 3; do PPCG_FP64_EMU=0 timeout 1200 python tools/time_to_solution.py $c >> gpurun_out/tts_r02_dmma.jsonl 2>> gpurun_out/tts_r02.err; done
timeout 600 python tools/iter_breakdown.py 3 3 5 > gpurun_out/breakdown3_r02.log 2>&1
