# driver protocol: reference arm then the repo arm with --steps 20 --warmup 5 (must finish < 1800 s)
( time timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
( time timeout 1790 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
tail -4 gpurun_out/r02_bench.err
