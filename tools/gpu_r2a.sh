set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.txt 2>&1
STORM_N=100000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists" \
    -s 6 -c 3 -o $OUT/full_c3 python tools/ncu_target.py c3 3 > $OUT/full_c3.log 2>&1
timeout 600 python bench.py --no-e2e > $OUT/bench.json 2> $OUT/bench.err
ls -la $OUT
