set -x
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_world.py tests/test_gpu_sharded.py -x -q > $OUT/fx3_tests.txt 2>&1
timeout 900 python tools/variants.py run c3,c2b rk prod > $OUT/fx3_var.txt 2>&1
STORM_N=100000000 timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_scan|k_finalize" -c 4 --csv python tools/ncu_target.py c3 2 > $OUT/fx3_ncu_c3.csv 2>&1
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_scan|k_finalize" -c 4 --csv python tools/ncu_target.py c2b 2 > $OUT/fx3_ncu_c2b.csv 2>&1
