for cfg in "8 256" "4 256" "3 128" "4 128" "6 128"; do set -- $cfg
echo "stages $1 nt $2"
SR_GEMM_STAGES=$1 SR_GEMM_NT_MAX=$2 timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 --max-tokens 1024 --reps 3 2>&1 | tail -1 | cut -c1-140
SR_GEMM_STAGES=$1 SR_GEMM_NT_MAX=$2 timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 80 --reps 3 2>&1 | tail -1 | cut -c1-140
done
