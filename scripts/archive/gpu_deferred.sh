timeout 900 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20
run() { w=$1; shift; env $E timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$E $w $*', round(d['ms_per_step'],4), 'tok/s %.4g' % d['value'], 'roof %.0f %.3f' % (r['achieved'], r['frac']))"; }
for c in 1 2 3; do E="TBA_SINGLE_CFG=$c"; run qwen_shard --schedule deferred; done
E=""; for w in rhomath pythia redteam; do run $w --schedule deferred; done
for c in 2 3; do
TBA_SINGLE_CFG=$c ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 1 --csv --log-file gpurun_out/dram_deferred_c$c.csv python bench.py --schedule deferred --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python -c "
import csv; r=list(csv.reader(open('gpurun_out/dram_deferred_c$c.csv'))); h=[x for x in r if x and x[0]=='ID'][0]
for x in r:
    if x and x[0]!='ID' and len(x)==len(h): d=dict(zip(h,x)); print('cfg $c', d['Metric Name'], d['Metric Value'])"
done
