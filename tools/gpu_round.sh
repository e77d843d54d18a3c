timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log | cut -c1-1500
timeout 1200 python bench.py --pair 1.5b+32b --budget 8192 --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
tail -3 gpurun_out/bench_c3.log | cut -c1-1500
