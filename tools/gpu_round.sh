for phi in 0 1; do
echo "phi $phi"
SR_ATTN_PHI=$phi timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullwidth.py -x -q -s 2>&1 | grep -E "prefill max|passed|failed" | head -4
SR_ATTN_PHI=$phi timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 80 2>&1 | tail -1 | cut -c1-100
SR_ATTN_PHI=$phi timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 --max-tokens 1024 --reps 3 2>&1 | tail -1 | cut -c1-100
done
