mkdir -p gpurun_out
for dn in 1.0 2.0; do
for m in qwen2.5-7b qwq-32b; do
  timeout 900 python tools/calibrate_judge.py $m --gpu --n 32 --cot-step 120 --iters 3 --digit-noise $dn > gpurun_out/calib_${m}_$dn.txt 2>&1
done
O7=$(grep OVERRIDE gpurun_out/calib_qwen2.5-7b_$dn.txt | cut -d' ' -f2)
O32=$(grep OVERRIDE gpurun_out/calib_qwq-32b_$dn.txt | cut -d' ' -f2)
timeout 600 python tools/loop_stats.py --pair 1.5b+7b --base-over "$O7" --steps 40 --problems 3 > gpurun_out/loop4_c2_$dn.txt 2>&1
timeout 900 python tools/loop_stats.py --pair 1.5b+32b --base-over "$O32" --steps 25 --problems 2 > gpurun_out/loop4_c3_$dn.txt 2>&1
done
