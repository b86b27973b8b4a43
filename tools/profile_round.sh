#!/bin/bash
# GPU-box profiling pass (run under gpurun from the repo root): the bench line, the launch list
# of the headline step, `ncu --set full` of the fault-path kernels (c2b) and of the storm's
# scan/finalize (c3, 2e7 entries), and of the translation and fold kernels.  Outputs land in
# gpurun_out/; tools/ncu_summary.py and tools/launch_summary.py turn them into profiles/.
set -x
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_c2b.csv \
    python bench.py --steps 2 --warmup 3 --no-storm --no-remap --no-e2e --no-check > $OUT/launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists|k_init|k_resolve|k_general" \
    -s 7 -c 7 -o $OUT/full_c2b python tools/ncu_target.py c2b 3 > $OUT/full_c2b.log 2>&1
STORM_N=20000000 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_finalize|k_lists" \
    -s 5 -c 3 -o $OUT/full_c3 python tools/ncu_target.py c3 2 > $OUT/full_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tr_" -s 6 -c 3 -o $OUT/full_tr \
    python tools/translate_run.py 3 > $OUT/full_tr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fold" -s 10 -c 5 -o $OUT/full_fold \
    python tools/fold_run.py 3 > $OUT/full_fold.log 2>&1
ls -la $OUT
