for c in torch lib; do
PYTHONFAULTHANDLER=1 PASTILA_COMM=$c timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 1 --warmup 1 --grid 256,512 --no-cpu-baseline --force-dist > gpurun_out/bench_fd_$c.json 2> gpurun_out/bench_fd_$c.err; echo "$c rc=$?"; head -c 200 gpurun_out/bench_fd_$c.json; echo
grep -v "NCCL INFO" gpurun_out/bench_fd_$c.err | grep -E "File \"/root|File \"/tmp|line|munmap|Error" | head -8
done
