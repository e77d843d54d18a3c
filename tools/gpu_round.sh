set -x
for m in r1-1.5b qwen2.5-7b; do
timeout 300 python tools/mk_prof.py $m --ctx 2048 > gpurun_out/mkprof_$m.log 2>&1
SR_MK_EVICT_FIRST=0 timeout 300 python tools/mk_prof.py $m --ctx 2048 > gpurun_out/mkprof_noef_$m.log 2>&1
done
cat gpurun_out/mkprof_*.log
