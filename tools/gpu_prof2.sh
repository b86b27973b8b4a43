OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan|k_finalize" -s 4 -c 2 -o $OUT/prof2_c2b python tools/ncu_target.py c2b 3 > $OUT/prof2_c2b.log 2>&1
STORM_N=100000000 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan|k_finalize" -s 4 -c 2 -o $OUT/prof2_c3 python tools/ncu_target.py c3 3 > $OUT/prof2_c3.log 2>&1
