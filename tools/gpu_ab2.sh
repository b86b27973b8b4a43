# parity tests of the current build, an A/B of build/var variants ($VARIANTS), and the ncu
# instruction / issue / traffic metrics of the current build's passes at c3 (2e7-entry prefix)
set -x
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-ab}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_world.py tests/test_gpu_sharded.py tests/test_gpu_trace.py -x -q > $OUT/${TAG}_tests.txt 2>&1
timeout 900 python tools/variants.py run c3,c2b ${VARIANTS:-base new} > $OUT/${TAG}_var.txt 2>&1
STORM_N=20000000 timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_scan|k_finalize|k_lists" -s 3 -c 3 --csv python tools/ncu_target.py c3 2 > $OUT/${TAG}_ncu_c3.csv 2>&1
ls -la $OUT
