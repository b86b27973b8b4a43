# parity tests of the current build, then an A/B of build/var variants ($VARIANTS, default "base new")
set -x
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-ab}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_world.py tests/test_gpu_sharded.py tests/test_gpu_trace.py -x -q > $OUT/${TAG}_tests.txt 2>&1
timeout 900 python tools/variants.py run c3,c2b ${VARIANTS:-base new} > $OUT/${TAG}_var.txt 2>&1
ls -la $OUT
