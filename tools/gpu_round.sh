timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 80 > gpurun_out/vp7b.log 2>&1
timeout 300 python tools/verify_profile.py r1-1.5b --ctx 2048 --m 80 > gpurun_out/vp15b.log 2>&1
timeout 300 python tools/verify_profile.py qwen2.5-7b --ctx 2048 --m 640 > gpurun_out/vp7b640.log 2>&1
cat gpurun_out/vp7b.log gpurun_out/vp15b.log gpurun_out/vp7b640.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
