#!/bin/bash
# A/B of the prefill attention kernels (scratch driver for gpurun)
mkdir -p gpurun_out
SR_ATTN=umma timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullwidth.py -x -q 2>&1 | tail -15 > gpurun_out/umma_tests.log
for a in ${ARMS:-tc umma}; do
  for m in ${MS:-80 640}; do
    SR_ATTN=$a timeout 120 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m $m --max-tokens 1024 --reps 5 2>&1 | tail -1 | sed "s/^/$a /"
  done
done > gpurun_out/umma_ab.log
if [ -n "$NCU" ]; then
SR_ATTN=umma timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vp_umma.csv python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 --max-tokens 1024 --reps 1 > /dev/null 2>&1
fi
cat gpurun_out/umma_tests.log gpurun_out/umma_ab.log
