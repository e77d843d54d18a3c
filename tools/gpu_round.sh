timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for m in r1-1.5b qwen2.5-7b qwq-32b; do
timeout 300 python tools/mk_prof.py $m --ctx 2048 > gpurun_out/mkprof_$m.log 2>&1
done
