# A/B of the COMBINE item width (SR_MK_COMBW=0: 32-dim items, 1: 64-dim).
# Usage: bash tools/combw_ab.sh [models...]; appends to gpurun_out/combw_ab.jsonl
mkdir -p gpurun_out
models=${@:-qwq-32b}
for rnd in 1 2; do
  for m in $models; do
    for ctx in 2048 6144; do
      for w in 0 1; do
        r=$(SR_MK_COMBW=$w timeout 600 python tools/decode_profile.py $m --ctx $ctx --new 48 --reps 2 2>&1 | tail -1)
        echo "{\"round\": $rnd, \"combw\": $w, \"res\": $r}" >> gpurun_out/combw_ab.jsonl
      done
    done
  done
done
