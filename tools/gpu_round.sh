timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/bench.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
