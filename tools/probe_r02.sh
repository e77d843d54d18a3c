# Round-2 GPU probe: the -m gpu suite, smoke, the default bench and its reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
SR_PARITY_REPORT=gpurun_out/parity_full_depth.jsonl timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=15 > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --spec-gamma 5 --no-cpu-baseline > gpurun_out/bench_g5.json 2> gpurun_out/bench_g5.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
