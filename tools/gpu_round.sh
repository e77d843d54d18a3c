for c in 2 1; do
SR_GEMM_CTAS_PER_SM=$c timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 80 2>&1 | tail -1 | cut -c1-110
SR_GEMM_CTAS_PER_SM=$c timeout 300 python tools/verify_profile.py r1-1.5b --ctx 2048 --m 80 2>&1 | tail -1 | cut -c1-110
SR_GEMM_CTAS_PER_SM=$c timeout 300 python tools/verify_profile.py qwq-32b --ctx 2048 --m 80 2>&1 | tail -1 | cut -c1-110
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
