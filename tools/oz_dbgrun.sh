mkdir -p gpurun_out
for d in 0 1 2 3 4 5 6; do echo "dbg=$d" >> gpurun_out/ozdbg.log; PPCG_OZ_DBG=$d timeout 120 python tools/oz_bench.py 2>&1 | grep tsgemm >> gpurun_out/ozdbg.log; done
