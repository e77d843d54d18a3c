timeout 1200 python bench.py --verify-template v2 --no-cpu-baseline > gpurun_out/bench_v2.log 2>&1
tail -1 gpurun_out/bench_v2.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['loop'])"
