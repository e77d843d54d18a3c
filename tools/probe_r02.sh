mkdir -p gpurun_out bench_data
set -x
timeout 900 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --dump-trace bench_data/1.5b+32b_trace.json > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python tools/measure_floors.py --out gpurun_out/floors.json > gpurun_out/floors.log 2>&1 && cp gpurun_out/floors.json tests/golden/floors.json
SR_PARITY_REPORT=gpurun_out/parity_report.jsonl timeout 1500 python -m pytest tests/test_gpu_trajectory_parity.py -x -q -s > gpurun_out/parity.log 2>&1
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cp bench_data/1.5b+32b_trace.json gpurun_out/
