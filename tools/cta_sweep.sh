# Persistent decode kernel: ms/token vs CTA count (SR_MK_CTAS, read when the
# model's workspace is sized).  Usage: bash tools/cta_sweep.sh model [ctas...]
# appends to gpurun_out/cta_sweep.jsonl
mkdir -p gpurun_out
m=${1:-r1-1.5b}; shift
for c in ${@:-148 132 116 100 84}; do
  for ctx in 2048 6144; do
    r=$(SR_MK_CTAS=$c timeout 600 python tools/decode_profile.py $m --ctx $ctx --new 48 --reps 2 2>&1 | tail -1)
    echo "{\"ctas\": $c, \"res\": $r}" >> gpurun_out/cta_sweep.jsonl
  done
done
