timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in r1-1.5b qwen2.5-7b qwq-32b; do
timeout 600 python tools/mk_prof.py $m --ctx 2048 > gpurun_out/mkprof_$m.log 2>&1
done
timeout 600 ncu --set full -k regex:decode_mk -c 1 -o gpurun_out/mk_7b python tools/decode_profile.py qwen2.5-7b --ctx 2048 --new 8 --reps 1 > gpurun_out/ncu_mk7b.log 2>&1
tail -1 gpurun_out/ncu_mk7b.log
