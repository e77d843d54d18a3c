timeout 600 python -m pytest tests/test_gpu_specdecode.py -x -q -s 2>&1 | tail -8
