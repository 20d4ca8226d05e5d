"""One LM-head fwd + bwd on a workload (for ncu launch lists of the backward kernels)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_18929_b200 as tba  # noqa: E402
import tba_synth as syn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="qwen_shard")
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--one-call", action="store_true")
ap.add_argument("--cublas", action="store_true", help="time the three cuBLAS GEMMs of the unfused path instead")
a = ap.parse_args()
w = syn.WORKLOADS[a.workload]
N, T, V, d = w.N, w.T, w.V, w.d
gi = syn.group_inputs(w, 0, 0, w.B)
hidden = torch.empty((N, T, d), dtype=torch.bfloat16, device="cuda")
weight = torch.empty((V, d), dtype=torch.bfloat16, device="cuda")
syn.fill_bf16_cuda(hidden.view(N * T, d), 0, "hidden", 0)
syn.fill_bf16_cuda(weight, 0, "weight", 0)
tok, mask = torch.from_numpy(gi["tokens"]).cuda(), torch.from_numpy(gi["mask"]).cuda()
ref, rew = torch.from_numpy(gi["ref_logp"]).cuda(), torch.from_numpy(gi["log_reward"]).cuda()
bws = torch.empty(tba.lmhead_bwd_workspace_bytes(N, T, d, V, a.chunk), dtype=torch.uint8, device="cuda")
dh = torch.empty((N, T, d), dtype=torch.bfloat16, device="cuda")
dw = torch.empty((V, d), dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
fw, bw = [], []
if a.cublas:
    rows = N * T
    lg = torch.empty((rows, V), dtype=torch.bfloat16, device="cuda")
    dhu = torch.empty((rows, d), dtype=torch.bfloat16, device="cuda")
    dwu = torch.empty((V, d), dtype=torch.bfloat16, device="cuda")
    for _ in range(a.reps):
        ev[0].record()
        torch.matmul(hidden.view(rows, d), weight.T, out=lg)
        ev[1].record()
        torch.matmul(lg, weight, out=dhu)
        torch.matmul(lg.T, hidden.view(rows, d), out=dwu)
        ev[2].record()
        torch.cuda.synchronize()
        fw.append(ev[0].elapsed_time(ev[1]))
        bw.append(ev[1].elapsed_time(ev[2]))
    print(f"cublas: logits {sorted(fw)[len(fw) // 2]:.1f} ms, dH+dW {sorted(bw)[len(bw) // 2]:.1f} ms")
    sys.exit(0)
fbws = torch.empty(tba.lmhead_fwd_bwd_workspace_bytes(N, T, d, V, w.K), dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    if a.one_call:
        ev[0].record()
        o = tba.lmhead_vargrad_fwd_bwd(hidden, weight, tok, mask, ref, rew, w.beta, w.K, N, dhidden=dh, dweight=dw,
                                       bwd_workspace=fbws)[0]
        ev[1].record()
        ev[2].record()
        torch.cuda.synchronize()
        fw.append(ev[0].elapsed_time(ev[1]))
        bw.append(0.0)
        continue
    ev[0].record()
    o, ws = tba.lmhead_vargrad_fwd(hidden, weight, tok, mask, ref, rew, w.beta, w.K, N)
    ev[1].record()
    tba.lmhead_vargrad_bwd(hidden, weight, tok, mask, ws, o.resid, 2.0 / N, dhidden=dh, dweight=dw,
                           chunk_rows=a.chunk, bwd_workspace=bws)
    ev[2].record()
    torch.cuda.synchronize()
    fw.append(ev[0].elapsed_time(ev[1]))
    bw.append(ev[1].elapsed_time(ev[2]))
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("TBA_"))
print(f"{a.workload} chunk={a.chunk} {env}: fwd {sorted(fw)[len(fw) // 2]:.1f} ms bwd {sorted(bw)[len(bw) // 2]:.1f} ms "
      f"(all bwd {[round(x, 1) for x in bw]}) loss {float(o.partial[0]):.6g}")
