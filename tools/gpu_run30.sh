timeout 3000 python tools/c4_run.py > gpurun_out/r02_c4.txt 2>&1; tail -3 gpurun_out/r02_c4.txt
