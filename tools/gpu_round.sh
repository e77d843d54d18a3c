timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullwidth.py -x -q 2>&1 | tail -1
timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 --max-tokens 1024 --reps 3 2>&1 | tail -1 | cut -c1-130
timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 80 2>&1 | tail -1 | cut -c1-90
timeout 300 python tools/decode_profile.py qwen2.5-7b --ctx 2048 --new 8 --reps 2 2>&1 | tail -1 | cut -c1-200
