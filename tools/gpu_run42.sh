python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_final.log 2>&1; tail -2 gpurun_out/gpu_tests_final.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo rc=$?; tail -c 3000 gpurun_out/bench_final.json
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; tail -c 1500 gpurun_out/bench_ref_final.json
