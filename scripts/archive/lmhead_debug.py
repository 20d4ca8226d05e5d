"""Quick GPU check of the LM-head-fused forward against a float64 torch reference (debug aid;
the parity tests against the oracle live in tests/test_gpu_lmhead.py)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2503_18929_b200 as tba  # noqa: E402


def ref_tok_lp(H, W, tok, inv_temp=1.0):
    z = (H.double().cpu().reshape(-1, H.shape[-1]) @ W.double().cpu().T) * inv_temp
    lse = torch.logsumexp(z, dim=1)
    return z.gather(1, tok.cpu().reshape(-1, 1)).squeeze(1) - lse


def case(N, T, d, V, integer, seed=0, inv_temp=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    if integer:
        H = (torch.randint(-2, 3, (N, T, d), generator=g).float() / 4).bfloat16()
        W = (torch.randint(-2, 3, (V, d), generator=g).float() / 4).bfloat16()
    else:
        H = torch.randn(N, T, d, generator=g).bfloat16()
        W = (torch.randn(V, d, generator=g) * (2.0 / d ** 0.5)).bfloat16()
    tok = torch.randint(0, V, (N, T), generator=g)
    mask = torch.ones(N, T, dtype=torch.uint8)
    Hd, Wd, td, md = H.cuda(), W.cuda(), tok.cuda(), mask.cuda()
    ws = torch.zeros(tba.lmhead_workspace_bytes(N, T, V), dtype=torch.uint8, device="cuda")
    out, nt = tba.lmhead_seq_logprob(Hd, Wd, td, md, inv_temp=inv_temp, workspace=ws, check_status=True)
    torch.cuda.synchronize()
    rows = N * T
    off = ((rows * 8 + 255) // 256) * 256
    lp = ws[off: off + rows * 8].view(torch.float64).cpu()
    ref = ref_tok_lp(H, W, tok, inv_temp)
    err = (lp - ref).abs()
    print(f"N={N} T={T} d={d} V={V} int={integer}: max|lp err| {err.max().item():.3e} at row {err.argmax().item()}"
          f" (lp {lp[err.argmax()].item():.6f} ref {ref[err.argmax()].item():.6f});"
          f" seq err {(out.cpu() - ref.view(N, T).sum(1)).abs().max().item():.3e}; nan rows {torch.isnan(lp).sum().item()}",
          flush=True)


def timing():
    N, T, d, V = 64, 1024, 3584, 152064
    H = torch.randn(N, T, d, device="cuda").bfloat16()
    W = (torch.randn(V, d, device="cuda") * (2.0 / d ** 0.5)).bfloat16()
    tok = torch.randint(0, V, (N, T), device="cuda")
    mask = torch.ones(N, T, dtype=torch.uint8, device="cuda")
    ws = torch.empty(tba.lmhead_workspace_bytes(N, T, V), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        tba.lmhead_seq_logprob(H, W, tok, mask, workspace=ws, check_status=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        tba.lmhead_seq_logprob(H, W, tok, mask, workspace=ws, check_status=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    fl = 2.0 * N * T * V * d
    print(f"fused lmhead fwd: {ms:.2f} ms  {fl / ms / 1e9:.0f} TFLOP/s", flush=True)
    logits = torch.empty(N, T, V, dtype=torch.bfloat16, device="cuda")
    for _ in range(2):
        torch.matmul(H.view(-1, d), W.T, out=logits.view(-1, V))
        tba.seq_logprob(logits, tok, mask, check_status=False)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        torch.matmul(H.view(-1, d), W.T, out=logits.view(-1, V))
    b.record()
    torch.cuda.synchronize()
    mm = a.elapsed_time(b) / 3
    a.record()
    for _ in range(3):
        torch.matmul(H.view(-1, d), W.T, out=logits.view(-1, V))
        tba.seq_logprob(logits, tok, mask, check_status=False)
    b.record()
    torch.cuda.synchronize()
    both = a.elapsed_time(b) / 3
    print(f"cuBLAS matmul (logits written): {mm:.2f} ms {fl / mm / 1e9:.0f} TFLOP/s; + seq_logprob: {both:.2f} ms",
          flush=True)


if __name__ == "__main__":
    case(1, 1, 64, 256, True)
    case(1, 128, 64, 256, True)
    case(3, 100, 256, 1000, True)
    case(2, 77, 1024, 50257, True, seed=1)
    case(2, 64, 3584, 152064, False, seed=2)
    case(2, 50, 3584, 152064, False, seed=3, inv_temp=1 / 0.7)
    if "--time" in sys.argv:
        timing()
