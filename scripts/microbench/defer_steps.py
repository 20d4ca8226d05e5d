"""Per-call times of the deferred pass over 30 back-to-back calls at the Qwen shard, on the bench's
synthetic logits and on randn*2 logits (developer probe: is the bench/ncu gap data or duration?)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_18929_b200 as tba  # noqa: E402
import tba_synth as syn  # noqa: E402

w = syn.WORKLOADS["qwen_shard"]
B, K, T, V = w.B, w.K, w.T, w.V
N = B * K
gi = syn.group_inputs(w, 0, 0, B)
lg = torch.empty((N, T, V), dtype=torch.bfloat16, device="cuda")
tok = torch.from_numpy(gi["tokens"]).cuda()
mk = torch.from_numpy(gi["mask"]).cuda()
rf = torch.from_numpy(gi["ref_logp"]).cuda()
rw = torch.from_numpy(gi["log_reward"]).cuda()
G = torch.empty_like(lg)
ws = torch.empty(tba.workspace_bytes(N, T), dtype=torch.uint8, device="cuda")
out = tba.ops._Fwd(N, K, torch.device("cuda"))
print("valid rows", int(gi["mask"].sum()), "of", N * T)
for name in ["synthetic", "randn", "synthetic"]:
    if name == "synthetic":
        syn.fill_logits_cuda(lg, 0, 0, V)
    else:
        g = torch.Generator(device="cuda").manual_seed(1)
        for i in range(N):
            lg[i] = (torch.randn(T, V, device="cuda", generator=g) * 2).to(torch.bfloat16)
    for gap in [0.0, 0.05]:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
        torch.cuda.synchronize()
        for a, b in evs:
            a.record()
            tba.vargrad_fwd_deferred(lg, tok, mk, rf, rw, w.beta, K, float(N), workspace=ws, out=out,
                                     grad_unscaled=G, check_status=False)
            b.record()
            if gap:
                torch.cuda.synchronize()
                time.sleep(gap)
        torch.cuda.synchronize()
        t = [a.elapsed_time(b) for a, b in evs]
        print(name, "sleep", gap, " ".join(f"{x:.3f}" for x in t))
