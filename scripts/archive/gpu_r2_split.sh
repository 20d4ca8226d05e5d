# A/B: deferred pass with the row split over a cluster of CS CTAs (contiguous parts, each part's
# first 96 KB on chip) vs the product (one 512-thread CTA per row).
mkdir -p gpurun_out
python scripts/ab_variants.py cs2=TBA_DEFER_CS=2 cs4=TBA_DEFER_CS=4 > /dev/null 2>&1
for v in cs2 cs4; do
TBA_LIBRARY=/tmp/tba_variants/$v/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k deferred 2>&1 | tail -1
done
for rep in 1 2; do
for v in prod cs2 cs4; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard pythia_fp32; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/sp_${v}_$wl.json 2>gpurun_out/sp_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/sp_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sp_${v}_$wl.err
  done
done
done
for v in prod cs2 cs4; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  TBA_LIBRARY=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:row_s -s 6 -c 1 --csv --log-file gpurun_out/sp_dram_$v.csv python bench.py --no-e2e --no-cpu-baseline --no-variants --schedule deferred --steps 2 --warmup 3 > /dev/null 2>&1
  grep -E "dram__|gpu__time" gpurun_out/sp_dram_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
