# Round-2 GPU probe: the -m gpu suite, smoke, the default bench (recording the
# reference arm's trace), the reference arm over that trace, and both arms as
# the driver runs them (--steps 20 --warmup 5).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
SR_PARITY_REPORT=gpurun_out/parity_full_depth.jsonl timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=10 > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --dump-trace gpurun_out/trace_bench.json > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --trace gpurun_out/trace_bench.json > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/driver_ref.json 2>> gpurun_out/bench_ref.err
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/driver_ours.json 2>> gpurun_out/bench.err
