timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; python -c "import json; d=json.load(open('gpurun_out/bench_r02b.json')); print(d['seconds_per_sweep'], d['e2e']['seconds'], d['m_best'], d['certification']['per_step'])"
