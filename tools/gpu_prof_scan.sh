OUT=gpurun_out
mkdir -p $OUT
STORM_N=100000000 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan" -s 2 -c 1 -o $OUT/prof_scan_c3 python tools/ncu_target.py c3 3 > $OUT/prof_scan_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan|k_finalize" -s 4 -c 2 -o $OUT/prof_c2b python tools/ncu_target.py c2b 3 > $OUT/prof_c2b.log 2>&1
