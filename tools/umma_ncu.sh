#!/bin/bash
mkdir -p gpurun_out
for a in tc umma; do
SR_ATTN=$a timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vp_$a.csv python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 --max-tokens 1024 --reps 1 > /dev/null 2>&1
done
ls -la gpurun_out
