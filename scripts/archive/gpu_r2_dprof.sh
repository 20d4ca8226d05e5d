# Deferred pass at the Qwen shard: phase trace (TBA_AB_DEFER_TRACE build) + ncu --set full of row_single1
mkdir -p gpurun_out
python scripts/ab_variants.py trace=TBA_AB_DEFER_TRACE > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/trace/libtba.so timeout 600 python scripts/defer_trace.py
ncu --set full --clock-control none --import-source on -k regex:row_single -s 3 -c 1 -o gpurun_out/prof_row_single_head -f python bench.py --no-e2e --no-cpu-baseline --no-variants --workload qwen_group --schedule deferred --steps 1 --warmup 3 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:row_single -s 2 -c 1 --csv --log-file gpurun_out/dram_deferred_head.csv python bench.py --no-e2e --no-cpu-baseline --no-variants --schedule deferred --steps 2 --warmup 3 > /dev/null 2>&1
tail -5 gpurun_out/dram_deferred_head.csv
