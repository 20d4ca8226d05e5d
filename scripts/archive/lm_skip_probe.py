"""Probe: does lmhead_fwd skip fully masked row blocks? Times full vs sparse masks."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2503_18929_b200 as tba  # noqa: E402

N, T, d, V = 16, 1024, 3584, 152064
H = torch.randn(N, T, d, device="cuda").bfloat16()
W = (torch.randn(V, d, device="cuda") * 0.03).bfloat16()
tok = torch.randint(0, V, (N, T), device="cuda")
ws = torch.empty(tba.lmhead_workspace_bytes(N, T, V), dtype=torch.uint8, device="cuda")
for name, L in (("full", T), ("quarter", T // 4), ("one block", 128), ("one row", 1)):
    mask = torch.zeros(N, T, dtype=torch.uint8, device="cuda")
    mask[:, :L] = 1
    for _ in range(2):
        tba.lmhead_seq_logprob(H, W, tok, mask, workspace=ws, check_status=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        tba.lmhead_seq_logprob(H, W, tok, mask, workspace=ws, check_status=False)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:10s} valid rows {int(mask.sum())}: {a.elapsed_time(b) / 3:.2f} ms", flush=True)
