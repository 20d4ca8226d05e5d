"""Summarise the ncu evidence brought back in gpurun_out/ into tracked files under profiles/.

    python scripts/ncu_summarize.py TAG

Reads gpurun_out/launches_TAG.csv (gpu__time_duration per launch, full Qwen shard),
gpurun_out/dram_TAG.csv (DRAM bytes per launch, full shard) and
gpurun_out/prof_<kernel>_TAG.ncu-rep (--set full on the one-group slice), and writes
profiles/TAG_summary.md plus profiles/ncu_traffic.json (traffic per launch for bench.py).
"""
import csv
import json
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def short(name):
    m = re.search(r"::(\w+)<", name) or re.search(r"(\w+)\(", name)
    base = m.group(1) if m else name[:40]
    return base


def read_metric_csv(path):
    rows = list(csv.reader(open(path)))
    h = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            out.append(dict(zip(h, r)))
    return out


def ncu_details(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if not rows:
        return {}, {}
    h = rows[0]
    ix = {n: i for i, n in enumerate(h)}
    det = {}
    for r in rows[1:]:
        det[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rawd = {}
    if len(rr) >= 3:
        for k, v in zip(rr[0], rr[2]):
            rawd[k] = v
    return det, rawd


def main(tag):
    os.makedirs(P, exist_ok=True)
    lines = [f"# ncu evidence, tag `{tag}`", "",
             "Commands: `scripts/gpu_profile.sh` (launch list and DRAM bytes on the full Qwen per-GPU shard "
             "driven by `bench.py`; `--set full` on the one-group slice `qwen_group`, same kernels and launch "
             "shape per row). ncu times are cold-cache and serialised: compare shares, not absolutes.", ""]
    lp = os.path.join(G, f"launches_{tag}.csv")
    if os.path.exists(lp):
        L = read_metric_csv(lp)
        by = {}
        for d in L:
            by.setdefault(short(d["Kernel Name"]), []).append(float(d["Metric Value"]))
        tot = sum(statistics.mean(v) for v in by.values())
        lines += ["## Launch list (gpu__time_duration, full shard)", "", "| kernel | launches | mean µs | share of step |",
                  "|---|---|---|---|"]
        for k, v in sorted(by.items(), key=lambda kv: -statistics.mean(kv[1])):
            lines.append(f"| {k} | {len(v)} | {statistics.mean(v) / 1e3:.1f} | {statistics.mean(v) / tot:.3f} |")
        lines.append("")
    dp = os.path.join(G, f"dram_{tag}.csv")
    traffic = {}
    traffic_lm = None
    if os.path.exists(dp):
        D = read_metric_csv(dp)
        agg = {}
        for d in D:
            k = short(d["Kernel Name"])
            agg.setdefault(k, {}).setdefault(d["Metric Name"], []).append(float(d["Metric Value"]))
        lines += ["## DRAM traffic per launch (full shard)", "", "| kernel | read GB | write GB | time µs | GB/s |",
                  "|---|---|---|---|---|"]
        for k, m in agg.items():
            r = statistics.mean(m.get("dram__bytes_read.sum", [0]))
            w = statistics.mean(m.get("dram__bytes_write.sum", [0]))
            t = statistics.mean(m.get("gpu__time_duration.sum", [1]))
            lines.append(f"| {k} | {r / 1e9:.3f} | {w / 1e9:.3f} | {t / 1e3:.1f} | {(r + w) / t:.0f} |")
            traffic[k] = r + w
        lines.append("")
    ddp = os.path.join(G, f"dram_deferred_{tag}.csv")
    if os.path.exists(ddp):  # the deferred-scale pass on the full shard (4V algorithmic bytes per valid row)
        D = read_metric_csv(ddp)
        agg = {}
        for d in D:
            agg.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"])
        alg = 65536 * 152064 * 2 * 2
        lines += ["## Deferred-scale pass `row_single1`, full Qwen shard (DRAM bytes per launch)", "",
                  "| launch | read GB | write GB | time µs | algorithmic 4V GB | algorithmic GB/s | DRAM GB/s |",
                  "|---|---|---|---|---|---|---|"]
        tot = []
        for k, m in agg.items():
            r, w, t = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"], m["gpu__time_duration.sum"]
            lines.append(f"| {k} | {r / 1e9:.2f} | {w / 1e9:.2f} | {t / 1e3:.0f} | {alg / 1e9:.2f} | {alg / t:.0f} | "
                         f"{(r + w) / t:.0f} |")
            tot.append(r + w)
        traffic["row_single"] = statistics.mean(tot)
        lines += ["", "Unique logits are 19.93 GB; reads above that are pass-2 re-reads that missed L2. ncu launches "
                  "are cold and alone; the bench's back-to-back steps run under the board power cap (DESIGN.md §5.4).", ""]
    lmp = os.path.join(G, f"lmhead_launches_{tag}.csv")
    if os.path.exists(lmp):
        M = read_metric_csv(lmp)
        agg = {}
        for d in M:
            agg.setdefault(short(d["Kernel Name"]), {}).setdefault(d["Metric Name"], []).append(float(d["Metric Value"]))
        tot = sum(statistics.mean(m.get("gpu__time_duration.sum", [0])) for m in agg.values()) or 1
        lines += ["## LM-head-fused forward (NEXT 3): launch list and DRAM bytes (full Qwen shard, "
                  "`bench.py --objective lmhead`)", "",
                  "| kernel | launches | mean µs | share of step | read GB | write GB |", "|---|---|---|---|---|---|"]
        for k, m in sorted(agg.items(), key=lambda kv: -statistics.mean(kv[1].get("gpu__time_duration.sum", [0]))):
            t = statistics.mean(m.get("gpu__time_duration.sum", [0]))
            r = statistics.mean(m.get("dram__bytes_read.sum", [0]))
            w = statistics.mean(m.get("dram__bytes_write.sum", [0]))
            lines.append(f"| {k} | {len(m.get('gpu__time_duration.sum', []))} | {t / 1e3:.1f} | {t / tot:.3f} | "
                         f"{r / 1e9:.3f} | {w / 1e9:.3f} |")
            if k == "lmhead_fwd":
                traffic_lm = r + w
        lines.append("")
    for rep in sorted(f for f in os.listdir(G) if f.startswith("prof_") and f.endswith(f"_{tag}.ncu-rep")):
        det, raw = ncu_details(os.path.join(G, rep))
        kname = rep[len("prof_"):-len(f"_{tag}.ncu-rep")]
        where = "full Qwen shard, bench --objective lmhead" if kname.startswith("lmhead") else "qwen_group slice"
        lines += [f"## `{kname}` — ncu --set full ({where})", ""]
        for key in ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
                    "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
                    "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "SM Frequency"]:
            if key in det:
                v, u = det[key]
                lines.append(f"- {key}: {v} {u}")
        for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                    "lts__t_sector_hit_rate.pct"]:
            if key in raw:
                lines.append(f"- {key}: {raw[key]}")
        stalls = []
        for k, v in raw.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        if stalls:
            tot = sum(s for s, _ in stalls) or 1
            top = ", ".join(f"{n} {s / tot:.0%}" for s, n in sorted(stalls, reverse=True)[:6])
            lines.append(f"- stall samples: {top}")
        lines.append("")
    open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    tp = os.path.join(P, "ncu_traffic.json")
    cur = json.load(open(tp)) if os.path.exists(tp) else {}
    if traffic_lm is not None:
        traffic["lmhead_fwd"] = traffic_lm
    if traffic:
        cur["qwen_shard"] = {**cur.get("qwen_shard", {}), **traffic}
        cur["_source"] = f"profiles/{tag}_summary.md (ncu dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        json.dump(cur, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1])
