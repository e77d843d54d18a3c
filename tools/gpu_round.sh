timeout 1500 python -m pytest tests/test_gpu_fullwidth.py -x -q -s 2>&1 | tail -15
timeout 300 python bench.py --mode tp --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
