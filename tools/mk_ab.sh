# A/B of the persistent decode kernel: ms/token and GB/s per model / context,
# with and without the weight stream (SR_MK_NOLOAD=1 times the consumer chain
# alone).  Usage: bash tools/mk_ab.sh [models...]; output gpurun_out/mk_ab.jsonl
mkdir -p gpurun_out
models=${@:-r1-1.5b qwen2.5-7b}
for m in $models; do
  for ctx in 2048 6144; do
    for nl in 0 1; do
      r=$(SR_MK_NOLOAD=$nl timeout 600 python tools/decode_profile.py $m --ctx $ctx --new 48 --reps 2 2>&1 | tail -1)
      echo "{\"noload\": $nl, \"res\": $r}" >> gpurun_out/mk_ab.jsonl
    done
  done
done
