"""Print an ncu --csv launch list (one row per launch, selected metrics as columns)."""
import csv
import io
import sys
from collections import OrderedDict

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
k = OrderedDict()
for r in csv.DictReader(io.StringIO(txt)):
    name = r["Kernel Name"]
    name = name.split("(")[0].replace("<unnamed>::", "").replace("tba::", "")[:34]
    k.setdefault((int(r["ID"]), name, r["Grid Size"]), {})[r["Metric Name"]] = r["Metric Value"].replace(",", "")
short = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc%",
         "sm__cycles_elapsed.avg.per_second": "clk", "lts__t_sector_hit_rate.pct": "L2hit%"}
for (i, n, g), m in k.items():
    print(f"{i:3d} {n:34s} {g:14s} " + " ".join(f"{short.get(a, a[:10])}={b}" for a, b in m.items()))
