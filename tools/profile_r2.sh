#!/bin/bash
# Round-2 evidence pass (run under gpurun from the repo root): the GPU test suite, the bench line,
# the reference arm, the launch list of the headline step, ncu --set full of the fault path at
# c3 (the whole 10^8-entry storm) and c2b, and of the fold's bucketed path.  Outputs: gpurun_out/${TAG}_*.
set -x
OUT=gpurun_out; TAG=${TAG:-r2}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/${TAG}_tests.txt 2>&1
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $OUT/${TAG}_ref.json 2> $OUT/${TAG}_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/${TAG}_launches_c2b.csv \
    python bench.py --steps 2 --warmup 3 --no-storm --no-remap --no-e2e --no-check > $OUT/${TAG}_launch_bench.log 2>&1
STORM_N=100000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists" \
    -s 3 -c 3 -o $OUT/${TAG}_full_c3 python tools/ncu_target.py c3 2 > $OUT/${TAG}_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists|k_init|k_resolve|k_general" \
    -s 7 -c 7 -o $OUT/${TAG}_full_c2b python tools/ncu_target.py c2b 3 > $OUT/${TAG}_full_c2b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fb_" -c 6 \
    -o $OUT/${TAG}_full_fold python tools/fold_run.py 1 > $OUT/${TAG}_full_fold.log 2>&1
ls -la $OUT | grep $TAG
