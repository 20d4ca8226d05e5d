"""Timeline of the forward row kernel (TBA_AB_FWD_TRACE build via TBA_LIBRARY): per row group start/end
(globaltimer), then the bandwidth-relevant shape: rows in flight over time, first start / last end,
time to drain the last 10 % of rows. Developer probe."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_18929_b200 as tba  # noqa: E402
import tba_synth as syn  # noqa: E402
from paper_2503_18929_b200 import _lib  # noqa: E402

for wl in sys.argv[1:] or ["pythia"]:
    w = syn.WORKLOADS[wl]
    B, K, T, V = w.B, w.K, w.T, w.V
    N = B * K
    gi = syn.group_inputs(w, 0, 0, B)
    lg = torch.empty((N, T, V), dtype=torch.bfloat16, device="cuda")
    syn.fill_logits_cuda(lg, 0, 0, V)
    tok = torch.from_numpy(gi["tokens"]).cuda()
    mk = torch.from_numpy(gi["mask"]).cuda()
    rf = torch.from_numpy(gi["ref_logp"]).cuda()
    rw = torch.from_numpy(gi["log_reward"]).cuda()
    ws = torch.empty(tba.workspace_bytes(N, T), dtype=torch.uint8, device="cuda")
    out = tba.ops._Fwd(N, K, torch.device("cuda"))
    for _ in range(4):
        tba.vargrad_fwd(lg, tok, mk, rf, rw, w.beta, K, float(N), workspace=ws, out=out, check_status=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tba.vargrad_fwd(lg, tok, mk, rf, rw, w.beta, K, float(N), workspace=ws, out=out, check_status=False)
    e1.record()
    torch.cuda.synchronize()
    L = _lib.load()
    rows = N * T
    buf = np.zeros(rows * 3, np.uint64)
    L.tba_debug_fwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
    assert L.tba_debug_fwd_trace(buf.ctypes.data, buf.size) == 0
    tr = buf.reshape(rows, 3).astype(np.int64)
    m = gi["mask"].reshape(-1) != 0
    tr = tr[m]
    sm, a, b = tr.T
    t0 = a.min()
    a = (a - t0) / 1e3
    b = (b - t0) / 1e3
    dur = b - a
    nbytes = m.sum() * V * 2
    print(f"{wl}: fwd+head event {e0.elapsed_time(e1)*1e3:.1f} us; rows {m.sum()}; first start 0, last start {a.max():.1f}, "
          f"last end {b.max():.1f} us; kernel-span GB/s {nbytes / (b.max() * 1e3):.0f}")
    print(f"  row duration us: p10 {np.percentile(dur,10):.1f} p50 {np.percentile(dur,50):.1f} p90 {np.percentile(dur,90):.1f} max {dur.max():.1f}")
    ends = np.sort(b)
    for q in (0.5, 0.9, 0.99, 1.0):
        print(f"  {q:.2f} of rows done by {ends[int(q * (len(ends) - 1))]:.1f} us")
    # rows in flight over time (10 us bins)
    grid = np.arange(0, b.max() + 10, 10.0)
    inflight = [(np.sum((a <= t) & (b > t))) for t in grid]
    print("  rows in flight per 10 us:", " ".join(str(x) for x in inflight))
