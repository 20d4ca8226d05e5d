"""Instruction histogram of one ncu --set full capture (source page, SASS): total warp instructions,
thread instructions per logit element, and the share by execution count (per-row vs per-element
work). Usage: python scripts/ncu_sass_hist.py REPORT.ncu-rep ELEMENTS [ROWS]"""
import collections
import csv
import io
import subprocess
import sys

rep, elems = sys.argv[1], float(sys.argv[2])
rows = float(sys.argv[3]) if len(sys.argv) > 3 else None
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
m = dict(zip(r[0], r[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]:
    print(f"{k:60s} {m.get(k)}")
rows_ = list(csv.reader(io.StringIO(src)))
h = rows_[1]
data = rows_[2:]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
cnt = [int(x[ia]) if x[ia].isdigit() else 0 for x in data]
tot = sum(cnt)
print(f"warp instructions {tot}, thread instructions per element {tot * 32 / elems:.2f}")
by = collections.Counter()
for c in cnt:
    by[c] += c
for c, s in sorted(by.items(), key=lambda x: -x[1])[:8]:
    extra = f" per row {c / rows:.2f}" if rows else ""
    print(f"  executed {c:>10d}x{extra}: share {s / tot:.3f} ({s // c if c else 0} instructions)")
