set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python tools/decode_profile.py qwen2.5-7b --ctx 2048 --new 32 > gpurun_out/dp7b.log 2>&1
timeout 600 python tools/decode_profile.py r1-1.5b --ctx 2048 --new 32 > gpurun_out/dp15b.log 2>&1
SR_DECODE=stream timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b.csv python tools/decode_profile.py qwen2.5-7b --ctx 2048 --new 8 --reps 1 > gpurun_out/ncu7b.log 2>&1
tail -3 gpurun_out/*.log
