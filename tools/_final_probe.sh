set -x
python -m pytest tests -m gpu -q -rs > gpurun_out/fin_gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo bench=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_bench_driver_args.json 2> gpurun_out/fin_bench_driver_args.err; echo bench20=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_ref_driver_args.json 2> gpurun_out/fin_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --kernel-name regex:sr:: -c 3000 --csv --log-file gpurun_out/fin_launches_c3.csv python bench.py --steps 4 --warmup 3 --windows 1 --ff-tokens 0 --no-cpu-baseline > gpurun_out/fin_ncu_bench.log 2>&1; echo ncu=$?
