mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_lmhead_bwd.py -x -q -k "pair or one_call" 2>&1 | tail -2
TBA_LMB_2SM=3 TBA_LMB_NT2=3 timeout 400 python -m pytest tests/test_gpu_lmhead_bwd.py -x -q 2>&1 | tail -2
for cfg in "0 0" "3 3" "1 1" "3 1" "0 0" "3 3" "1 1"; do set -- $cfg; TBA_LMB_2SM=$1 TBA_LMB_NT2=$2 timeout 300 python scripts/lm_bwd_probe.py --one-call --reps 4; done
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
TBA_LMB_2SM=3 TBA_LMB_NT2=3 timeout 300 ncu --metrics $M -k regex:tc_gemm -c 4 --clock-control none --csv --log-file gpurun_out/nt2.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
python scripts/ncu_table.py gpurun_out/nt2.csv
