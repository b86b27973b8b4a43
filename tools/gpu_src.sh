# source-level ncu capture of the fault-path passes (c3 prefix and c2b)
set -x
OUT=gpurun_out
mkdir -p $OUT
STORM_N=20000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_fx|k_finalize_fx|k_lists" -s 3 -c 3 -o $OUT/src_c3 python tools/ncu_target.py c3 2 > $OUT/src_c3.log 2>&1
ls -la $OUT
