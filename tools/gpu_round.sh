timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1
tail -1 gpurun_out/bench_default.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['breakdown_ms_per_step'], d['loop'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])"
