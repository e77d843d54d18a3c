timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k long 2>&1 | tail -3
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log | cut -c1-400
