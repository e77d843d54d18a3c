timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 > gpurun_out/bench_dp2.log 2>&1
tail -2 gpurun_out/bench_dp2.log | cut -c1-700
timeout 1500 python bench.py --pair 1.5b+32b --budget 8192 --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
tail -1 gpurun_out/bench_c3.log | cut -c1-1600
