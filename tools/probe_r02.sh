mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_c3.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mk -c 1 -o gpurun_out/r02_ncu_decode_mk_32b -f python tools/decode_profile.py qwq-32b --ctx 4096 --new 24 --reps 1 > gpurun_out/ncu_32b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mk -c 1 -o gpurun_out/r02_ncu_decode_mk_15b -f python tools/decode_profile.py r1-1.5b --ctx 4096 --new 24 --reps 1 > gpurun_out/ncu_15b.log 2>&1
