set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_keys.py -x -q 2>&1 | tail -30 > gpurun_out/keys_tests.log
cat gpurun_out/keys_tests.log
timeout 600 python bench.py --grid 64,256,512 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_grid3.json 2> gpurun_out/bench_grid3.err
tail -3 gpurun_out/bench_grid3.err; cat gpurun_out/bench_grid3.json
