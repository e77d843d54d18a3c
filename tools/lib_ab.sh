# Same-box A/B of two builds of the library (SR_LIB) and/or env knobs.
# Usage: bash tools/lib_ab.sh "<tag>=<env assignments>" ... ; appends to gpurun_out/lib_ab.jsonl
# e.g.   bash tools/lib_ab.sh "head=SR_LIB=build_ab/libhead.so" "split1=SR_MK_GUSPLIT=1"
mkdir -p gpurun_out
models=${MODELS:-r1-1.5b qwq-32b}
for rnd in 1 2; do
  for m in $models; do
    for ctx in 2048 6144; do
      for arm in "$@"; do
        tag=${arm%%=*}; envs=${arm#*=}
        r=$(env $envs timeout 600 python tools/decode_profile.py $m --ctx $ctx --new 48 --reps 2 2>&1 | tail -1)
        echo "{\"round\": $rnd, \"arm\": \"$tag\", \"res\": $r}" >> gpurun_out/lib_ab.jsonl
      done
    done
  done
done
