timeout 600 ncu --set full --import-source on -k regex:decode_mk -c 1 -o gpurun_out/mk_15b_v2 python tools/decode_profile.py r1-1.5b --ctx 2048 --new 16 --reps 1 > gpurun_out/ncu_mk15.log 2>&1
tail -1 gpurun_out/ncu_mk15.log
