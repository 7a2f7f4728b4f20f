python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_final.log 2>&1; tail -2 gpurun_out/gpu_tests_final.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo rc=$?; tail -c 400 gpurun_out/bench_final.json
python tools/c5_run.py > gpurun_out/r02_c5_final.txt 2>&1; tail -2 gpurun_out/r02_c5_final.txt
PASTILA_DEBUG=1 python tools/c4_run.py > gpurun_out/r02_c4_pruned.txt 2> gpurun_out/c4_err.log; cat gpurun_out/r02_c4_pruned.txt
