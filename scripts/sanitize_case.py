"""Small cases through the C ABI for compute-sanitizer (memcheck/racecheck/synccheck/initcheck).
Every buffer the kernels read is initialised; dlogits is allocated uninitialised so initcheck
proves that masked rows are written (zero-filled), and a second pass reads it back."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_18929_b200 as tba  # noqa: E402
import tba_synth as syn  # noqa: E402

cases = [
    dataclasses.replace(syn.WORKLOADS["toy"]),
    dataclasses.replace(syn.WORKLOADS["redteam"], B=2, K=3, T=5, len_lo=1, len_hi=5),    # unaligned, ragged
    dataclasses.replace(syn.WORKLOADS["rhomath"], B=2, K=4, T=6, V=4093, len_lo=0, len_hi=6),  # warp path
    dataclasses.replace(syn.WORKLOADS["qwen"], B=1, K=2, T=2),                              # long rows
]
for w in cases:
    gi = syn.group_inputs(w, 0, 0, w.B)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    lg = torch.empty((w.N, w.T, w.V), dtype=dt, device="cuda")
    syn.fill_logits_cuda(lg, 0, 0, w.V)
    tok = torch.from_numpy(gi["tokens"]).cuda()
    mask = torch.from_numpy(gi["mask"]).cuda()
    ref = torch.from_numpy(gi["ref_logp"]).cuda()
    rew = torch.from_numpy(gi["log_reward"]).cuda()
    ws = torch.empty(tba.workspace_bytes(w.N, w.T), dtype=torch.uint8, device="cuda")
    o, _ = tba.vargrad_fwd(lg, tok, mask, ref, rew, w.beta, w.K, float(w.N), workspace=ws, check_status=True)
    d = torch.empty_like(lg)
    tba.vargrad_bwd(lg, tok, mask, ws, o.resid, 2.0 / w.N, dlogits=d)
    sl, nt = tba.seq_logprob(lg, tok, mask, check_status=True)
    # the other entry points: TBA' (two-call and deferred), fused one-launch, deferred TB
    gen = torch.from_numpy(syn.gen_logp(w, 0)).cuda()
    ntok = float(max(int(mask.sum().item()), 1))
    ob, wsb = tba.tbap_fwd(lg, tok, mask, gen, ref, rew, w.beta, w.K, "icepop", 0.5, 2.0, ntok, check_status=True)
    db = tba.tbap_bwd(lg, tok, mask, wsb, ob.coef, ntok)
    G = torch.empty_like(lg)
    tba.tbap_fwd(lg, tok, mask, gen, ref, rew, w.beta, w.K, "clip", 0.0, 8.0, ntok, grad_unscaled=G)
    of, _, df, _ = tba.vargrad_fused(lg, tok, mask, ref, rew, w.beta, w.K, float(w.N), check_status=True)
    od, _, Gd = tba.vargrad_fwd_deferred(lg, tok, mask, ref, rew, w.beta, w.K, float(w.N), check_status=True)
    op, _, dp, _ = tba.vargrad_pipelined(lg, tok, mask, ref, rew, w.beta, w.K, float(w.N), groups_per_chunk=1,
                                         check_status=True)
    torch.cuda.synchronize()
    assert torch.equal(op.partial, o.partial) and torch.equal(dp, d)
    s2 = float(db.float().sum().item() + G.float().sum().item() + df.float().sum().item() + Gd.float().sum().item())
    s = float(d.float().sum().item())  # reads every dlogits element (initcheck)
    print(w.name, w.V, "loss", o.partial[0].item(), "sum dlogits", s, "seq_logprob match",
          torch.equal(sl, o.seq_logp), "other paths", s2, torch.equal(of.partial, o.partial))
# LM-head-fused forward (tcgen05 + TMA kernel): ragged rows / vocab / d tails
wl = dataclasses.replace(syn.WORKLOADS["toy"], B=2, K=4, T=37, V=1000, d=200, len_lo=0, len_hi=37)
gl = syn.group_inputs(wl, 2, 0, wl.B)
hid = torch.empty((wl.N, wl.T, wl.d), dtype=torch.bfloat16, device="cuda")
wt = torch.empty((wl.V, wl.d), dtype=torch.bfloat16, device="cuda")
syn.fill_bf16_cuda(hid.view(wl.N * wl.T, wl.d), 2, "hidden", 0)
syn.fill_bf16_cuda(wt, 2, "weight", 0)
ol, lws = tba.lmhead_vargrad_fwd(hid, wt, torch.from_numpy(gl["tokens"]).cuda(), torch.from_numpy(gl["mask"]).cuda(),
                               torch.from_numpy(gl["ref_logp"]).cuda(), torch.from_numpy(gl["log_reward"]).cuda(),
                               wl.beta, wl.K, float(wl.N), check_status=True)
# LM-head backward: two-call (GEMM recompute of dz, chunks of 128 rows) and one-call (stored logits)
dh, dw = tba.lmhead_vargrad_bwd(hid, wt, torch.from_numpy(gl["tokens"]).cuda(), torch.from_numpy(gl["mask"]).cuda(),
                                lws, ol.resid, 2.0 / wl.N, chunk_rows=128)
o1, dh1, dw1 = tba.lmhead_vargrad_fwd_bwd(hid, wt, torch.from_numpy(gl["tokens"]).cuda(),
                                          torch.from_numpy(gl["mask"]).cuda(), torch.from_numpy(gl["ref_logp"]).cuda(),
                                          torch.from_numpy(gl["log_reward"]).cuda(), wl.beta, wl.K, float(wl.N),
                                          groups_per_chunk=1, check_status=True)
torch.cuda.synchronize()
assert torch.equal(dh, dh1)
print("lmhead loss", ol.partial[0].item(), "dW sum", float(dw.sum().item()), float(dw1.sum().item()))
print("sanitize cases done")
