timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
timeout 1500 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_full_keys.json 2> gpurun_out/bench_full_keys.err
tail -2 gpurun_out/bench_full_keys.err; cat gpurun_out/bench_full_keys.json
