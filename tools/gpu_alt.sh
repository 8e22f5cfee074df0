# the alternative code paths still pass the device suite: DMMA products, digit cache off, Jacobi pencils
mkdir -p gpurun_out
PPCG_FP64_EMU=0 timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_ozaki_gpu.py --deselect tests/test_fullshape_kernels_gpu.py 2>&1 | tail -4 > gpurun_out/alt_dmma.log
PPCG_DIGIT_CACHE=0 timeout 1500 python -m pytest tests/test_solver_gpu.py tests/test_golden_gpu.py tests/test_distributed_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/alt_nocache.log
PPCG_PENCIL_EIG=jacobi timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_solver_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/alt_jacobi.log
