# cta_group::2 backward GEMM: DRAM reads per launch vs raster (ncu, 4 launches each)
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for cfg in "3 3 32" "3 0 32" "3 0 8" "3 0 64" "0 3 32" "0 0 32"; do
  set -- $cfg
  TBA_LMB_2SM=$1 TBA_LMB_NINNER=$2 TBA_LMB_SWZ=$3 timeout 300 ncu --metrics $M -k regex:tc_gemm -c 4 --clock-control none --csv --log-file gpurun_out/pr_$1_$2_$3.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
  echo "== 2SM=$1 NINNER=$2 SWZ=$3"; python scripts/ncu_table.py gpurun_out/pr_$1_$2_$3.csv
done
