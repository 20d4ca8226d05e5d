# NEXT 3 bench lines at the round-2 code: the LM-head-fused forward and the one-call training step
# (Qwen shard, RhoMath), with the interleaved cuBLAS comparisons.
mkdir -p gpurun_out
for wl in qwen_shard rhomath; do
  timeout 900 python bench.py --workload $wl --objective lmhead --no-e2e > gpurun_out/bench_r02_${wl}_lmhead.json 2>gpurun_out/bench_r02_${wl}_lmhead.err
  timeout 1200 python bench.py --workload $wl --objective lmhead_train --steps 10 --warmup 3 > gpurun_out/bench_r02_${wl}_lmtrain.json 2>gpurun_out/bench_r02_${wl}_lmtrain.err
done
python - <<'PY'
import json
for wl in ("qwen_shard", "rhomath"):
    for o in ("lmhead", "lmtrain"):
        try:
            d = json.loads(open(f"gpurun_out/bench_r02_{wl}_{o}.json").read().strip().splitlines()[-1])
        except Exception as e:
            print(wl, o, "ERR", e); continue
        v = d.get("variants", {})
        print(wl, o, round(d["ms_per_step"], 2), "TF/s", round(d["roofline"]["achieved"]), "frac", round(d["roofline"]["frac"], 3),
              {k: {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in x.items() if kk in ("ms_per_step", "fused_over_unfused", "fused_ms_paired")} for k, x in v.items()},
              d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
