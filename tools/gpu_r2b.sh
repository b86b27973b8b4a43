set -x
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_large_world.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_bench_multirank.py -x -q > $OUT/gpu_tests_new.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ls -la $OUT
