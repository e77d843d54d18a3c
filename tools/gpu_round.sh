timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullwidth.py tests/test_gpu_decode.py -x -q 2>&1 | tail -1
timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 --max-tokens 1024 --reps 3 2>&1 | tail -1 | cut -c1-130
for m in qwen2.5-7b r1-1.5b qwq-32b; do
timeout 300 python tools/verify_profile.py $m --ctx 2048 --m 80 2>&1 | tail -1 | cut -c1-90
done
