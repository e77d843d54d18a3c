timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py tests/test_gpu_fullwidth.py -m gpu -q -p no:cacheprovider 2>&1 | tail -8
for round in 1 2; do for v in 1 0; do SR_MK_TILED=$v MK_TAG="tiled$v" bash tools/mk_ab.sh qwq-32b qwen2.5-7b r1-1.5b; done; done
SR_MK_NOLOAD=1 MK_TAG=noload_tiled bash tools/mk_ab.sh qwq-32b r1-1.5b
