mkdir -p gpurun_out
PPCG_B200_LIB=$PWD/paper_1407_7506_b200/libppcg_b200_prof.so timeout 900 python tools/pencil_phases.py 5 3 64 512 > gpurun_out/pencil_phases5.txt 2>&1
PPCG_B200_LIB=$PWD/paper_1407_7506_b200/libppcg_b200_prof.so timeout 900 python tools/pencil_phases.py 3 3 > gpurun_out/pencil_phases3.txt 2>&1
