"""Phase trace of the deferred row pass (TBA_AB_DEFER_TRACE build, loaded through TBA_LIBRARY):
per row the SM and the SM clock at start / pass-1 register loop done / pass 1 done / pass 2
start / end; prints per-phase means and each SM's occupancy by phase. Developer tool."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_18929_b200 as tba  # noqa: E402
from paper_2503_18929_b200 import _lib  # noqa: E402

N, T, V, K = int(os.environ.get("TR_N", 64)), int(os.environ.get("TR_T", 1024)), int(os.environ.get("TR_V", 152064)), 8
g = torch.Generator(device="cuda").manual_seed(1)
lg = (torch.randn(N, T, V, device="cuda", generator=g) * 2).to(torch.bfloat16)
tk = torch.randint(0, V, (N, T), device="cuda", generator=g)
mk = torch.ones(N, T, dtype=torch.uint8, device="cuda")
rf = torch.zeros(N, dtype=torch.float64, device="cuda")
rw = torch.zeros(N, dtype=torch.float64, device="cuda")
G = torch.empty_like(lg)
for _ in range(3):
    tba.vargrad_fwd_deferred(lg, tk, mk, rf, rw, 1.0, K, float(N), grad_unscaled=G, check_status=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tba.vargrad_fwd_deferred(lg, tk, mk, rf, rw, 1.0, K, float(N), grad_unscaled=G, check_status=False)
e1.record()
torch.cuda.synchronize()
print("step ms", e0.elapsed_time(e1))
L = _lib.load()
rows = min(N * T, 1 << 17)
buf = np.zeros(rows * 6, np.uint64)
L.tba_debug_defer_trace.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
assert L.tba_debug_defer_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(rows, 6).astype(np.int64)
np.save("gpurun_out/defer_trace.npy", tr)
sm, t0, t1, t2, t3, t4 = tr.T
ghz = 1.965e3  # clocks per us at 1965 MHz
print("phase means (us): loads issued %.2f | pass1 rest %.2f | reduce+finalize %.2f | pass2 %.2f | total %.2f" % (
    np.mean(t1 - t0) / ghz, np.mean(t2 - t1) / ghz, np.mean(t3 - t2) / ghz, np.mean(t4 - t3) / ghz,
    np.mean(t4 - t0) / ghz))
for q in (10, 50, 90):
    print(f"p{q} pass1 %.2f pass2 %.2f total %.2f" % (np.percentile(t2 - t0, q) / ghz, np.percentile(t4 - t3, q) / ghz,
                                                 np.percentile(t4 - t0, q) / ghz))
# per SM: time-weighted count of CTAs in pass 1 / pass 2, and idle gaps between a CTA's end and the next start
occ = []
gaps = []
for s in np.unique(sm)[:148]:
    r = tr[sm == s]
    r = r[np.argsort(r[:, 1])]
    lo, hi = r[:, 1].min(), r[:, 5].max()
    ev = []
    for a in r:
        ev += [(a[1], 1, 0), (a[3], -1, 0), (a[4], 0, 1), (a[5], 0, -1)]
    ev.sort()
    p1 = p2 = 0
    last = lo
    hist = np.zeros((3, 3))
    for t, d1, d2 in ev:
        hist[min(p1, 2), min(p2, 2)] += t - last
        last = t
        p1 += d1
        p2 += d2
    occ.append(hist / (hi - lo))
    gaps.append(len(r))
occ = np.mean(occ, axis=0)
print("fraction of SM time with (#CTAs in pass 1 [rows], #CTAs in pass 2 [cols]):")
print(np.array2string(occ, precision=3))
print("rows per SM (mean)", np.mean(gaps))
