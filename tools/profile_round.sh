#!/bin/bash
# GPU-box profiling pass (run under gpurun): launch list of the headline bench command and one
# `ncu --set full` capture per hot kernel (c2b), plus the storm's scan/finalize (c3, 2e7 entries).
# Outputs land in gpurun_out/; tools/ncu_summary.py turns them into profiles/ summaries.
set -x
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c2b.csv \
    python bench.py --steps 2 --warmup 3 --no-storm --no-remap --no-e2e --no-check > $OUT/launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists|k_init|k_resolve" \
    -s 7 -c 5 -o $OUT/full_c2b python tools/ncu_target.py c2b 3 > $OUT/full_c2b.log 2>&1
STORM_N=20000000 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists" \
    -s 5 -c 3 -o $OUT/full_c3 python tools/ncu_target.py c3 2 > $OUT/full_c3.log 2>&1
ls -la $OUT
