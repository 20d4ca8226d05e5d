# Small shapes: bench lines and the ncu launch list (kernel durations, DRAM bytes) per workload
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for wl in pythia redteam gsm8k_t3 gsm8k_k40; do
  $B --workload $wl > gpurun_out/sm_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sm_$wl.json')); k=d['kernels']; print('$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 9 -c 3 --csv $B --workload $wl --steps 2 --warmup 3 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' -v w=$wl '{split($5,a,"<"); print w, a[1], $(NF-2), $NF}'
done
