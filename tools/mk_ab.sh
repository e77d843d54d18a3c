# Persistent decode kernel: ms/token and GB/s per model / context.
# Usage: bash tools/mk_ab.sh [models...]; appends to gpurun_out/mk_ab.jsonl
mkdir -p gpurun_out
models=${@:-r1-1.5b qwen2.5-7b}
for m in $models; do
  for ctx in 2048 6144; do
    r=$(timeout 600 python tools/decode_profile.py $m --ctx $ctx --new 48 --reps 2 2>&1 | tail -1)
    echo "{\"tag\": \"${MK_TAG:-}\", \"res\": $r}" >> gpurun_out/mk_ab.jsonl
  done
done
