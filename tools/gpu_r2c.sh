set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gpu_tests_c.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c.json 2> $OUT/bench_c.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref_c.json 2> $OUT/bench_ref_c.err
STORM_N=100000000 timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_scan|k_finalize|k_lists" -c 6 --csv python tools/ncu_target.py c3 2 > $OUT/ncu_c3_c.csv 2>&1
ls -la $OUT
