mkdir -p gpurun_out
PPCG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
PPCG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_2rank_ref.json 2> gpurun_out/bench_2rank_ref.err
timeout 900 python -m pytest tests/test_distributed_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/tests_dist.log
