"""GPU parity of the LM-head backward (NEXT 3; tba_lmhead_tb_loss_bwd / tba_lmhead_tbap_loss_bwd):
dL/dhidden and dL/dW against the fp64 oracle (oracle.lmhead_grads applied to the oracle's
dlogits of z = W h; pinned by finite differences in tests/test_oracle_lmhead.py).

Tolerance (reading R21). The kernels round dz to bf16 (round-to-nearest-even,
relative error <= 2^-9) before the two gradient GEMMs, which accumulate in fp32. With
A = |dZ| |W| (for dH) or |dZ|^T |H| (for dW), the oracle's fp64 exact dz gives, per element,
    |err| <= 2^-8 A + 4 sqrt(K) 2^-24 A + 1e-12
(2^-9 for the rounding doubled to cover the fp32 softmax in dz and the recomputed logits' fp32
accumulation error, which enters p relatively; the fp32 accumulation of the K-term sums,
K = V for dH and the chunk's rows for dW, by its statistical sqrt(K) growth, 4 sigma)."""
import dataclasses
import math

import numpy as np
import pytest

import tba_synth as syn
from oracle import tba_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2503_18929_b200 as tba  # noqa: E402


def W(name, **kw):
    return dataclasses.replace(syn.WORKLOADS[name], **kw)


def inputs(w, seed, kind):
    gi = syn.group_inputs(w, seed, 0, w.B)
    N, T, d, V = w.N, w.T, w.d, w.V
    hb = torch.empty((N, T, d), dtype=torch.bfloat16, device="cuda")
    wb = torch.empty((V, d), dtype=torch.bfloat16, device="cuda")
    syn.fill_bf16_cuda(hb.view(N * T, d), seed, "hidden", 0, kind)
    syn.fill_bf16_cuda(wb, seed, "weight", 0, kind)
    H = syn.bf16_bits_to_f64(syn.hidden_rows(seed, d, np.arange(N * T), kind))
    Wh = syn.bf16_bits_to_f64(syn.weight_rows(seed, d, np.arange(V), kind))
    dev = dict(hidden=hb, weight=wb, tokens=torch.from_numpy(gi["tokens"]).cuda(),
               mask=torch.from_numpy(gi["mask"]).cuda(), ref_logp=torch.from_numpy(gi["ref_logp"]).cuda(),
               log_reward=torch.from_numpy(gi["log_reward"]).cuda())
    return dev, gi, H, Wh


def check_grad(got, want, A, K, what):
    tol = (2.0 ** -8 + 4 * math.sqrt(K) * 2.0 ** -24) * A + 1e-12
    err = np.abs(got - want)
    bad = err > tol
    assert not bad.any(), (f"{what}: {bad.sum()} of {bad.size} outside the bound; worst err "
                           f"{err[bad].max():.3g} vs tol {tol[bad][np.argmax(err[bad])]:.3g}")
    return float(np.max(err / np.maximum(A, 1e-30)))


def oracle_grads(H, Wh, dz):
    dH, dW = O.lmhead_grads(H, Wh, dz)
    return dH, dW, np.abs(dz) @ np.abs(Wh), np.abs(dz).T @ np.abs(H)


CASES = [
    # name, workload, input kind, chunk_rows, inv_temp, dhidden dtype
    ("lattice_ragged_chunks", W("toy", B=2, K=4, T=40, V=1000, d=200, len_lo=0, len_hi=40), "lattice", 128, 1.0,
     torch.float32),
    ("normal_temp_bf16_dh", W("pythia", B=2, K=4, T=64, V=5000, d=128), "normal", 0, 1 / 0.7, torch.bfloat16),
    ("gpt2_odd_vocab", W("redteam", B=2, K=2, T=20, d=96), "normal", 256, 1.0, torch.float32),
    ("skipped_rows", W("rhomath", B=1, K=4, T=256, V=700, d=64, len_lo=0, len_hi=128), "lattice", 0, 1.0,
     torch.float32),
]


@pytest.mark.parametrize("name,w,kind,chunk,inv_temp,dh_dt", CASES, ids=[c[0] for c in CASES])
def test_lmhead_tb_bwd_parity(name, w, kind, chunk, inv_temp, dh_dt):
    dev, gi, H, Wh = inputs(w, 11, kind)
    N, T, V = w.N, w.T, w.V
    o, ws = tba.lmhead_vargrad_fwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], dev["ref_logp"],
                                   dev["log_reward"], w.beta, w.K, N, inv_temp=inv_temp, check_status=True)
    dh, dw = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.resid,
                                    2.0 / N, inv_temp=inv_temp, dhidden_dtype=dh_dt, chunk_rows=chunk)
    torch.cuda.synchronize()
    z = O.lmhead_logits(H, Wh).reshape(N, T, V)
    r = O.vargrad_head(z, gi["tokens"], gi["mask"], gi["ref_logp"], gi["log_reward"], w.beta, w.K,
                       inv_temp=inv_temp)
    dz = r["dlogits"].reshape(N * T, V)
    dH, dW, AH, AW = oracle_grads(H, Wh, dz)
    got_h = dh.double().cpu().numpy().reshape(N * T, -1)
    if dh_dt == torch.bfloat16:  # the stored value is the fp32 result rounded once more
        AH = AH + np.abs(dH) * 2.0 ** -8 / (2.0 ** -8 + 4 * math.sqrt(V) * 2.0 ** -24)
    check_grad(got_h, dH, AH, V, "dhidden")
    check_grad(dw.double().cpu().numpy(), dW, AW, max(chunk or N * T, 1), "dweight")
    # masked rows of dhidden are exactly zero
    m = gi["mask"].reshape(-1) == 0
    assert np.all(got_h[m] == 0.0)


def test_lmhead_bwd_learned_logz_accumulate_and_partial_outputs():
    w = W("pythia", B=2, K=4, T=24, V=3000, d=64)
    dev, gi, H, Wh = inputs(w, 12, "lattice")
    N, T, V = w.N, w.T, w.V
    log_z = torch.tensor([0.5, -1.25], dtype=torch.float64, device="cuda")
    o, ws = tba.lmhead_vargrad_fwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], dev["ref_logp"],
                                   dev["log_reward"], w.beta, w.K, N, log_z_param=log_z, check_status=True)
    g = torch.tensor(0.75, dtype=torch.float64, device="cuda")
    dh, dw, dlz = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.resid,
                                         2.0 / N, grad_out=g, log_z_param=log_z, K=w.K)
    # accumulate: a second call adds the same gradient
    dh2, dw2, _ = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.resid,
                                         2.0 / N, grad_out=g, log_z_param=log_z, K=w.K, dhidden=dh.clone(),
                                         dweight=dw.clone(), accumulate=True)
    # dweight only / dhidden only
    dh3, dw3, _ = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.resid,
                                         2.0 / N, grad_out=g, log_z_param=log_z, K=w.K, want_dhidden=False)
    dh4, dw4, _ = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.resid,
                                         2.0 / N, grad_out=g, log_z_param=log_z, K=w.K, want_dweight=False)
    torch.cuda.synchronize()
    assert dh3 is None and dw4 is None
    assert torch.equal(dw3, dw) and torch.equal(dh4, dh)
    torch.testing.assert_close(dh2, 2 * dh, rtol=1e-6, atol=0)
    torch.testing.assert_close(dw2, 2 * dw, rtol=1e-6, atol=0)
    z = O.lmhead_logits(H, Wh).reshape(N, T, V)
    r = O.vargrad_head(z, gi["tokens"], gi["mask"], gi["ref_logp"], gi["log_reward"], w.beta, w.K,
                       log_z=log_z.cpu().numpy(), grad_out=0.75)
    # per-group quantity: the north_star bar for per-sequence values (rel 1e-4, abs 1e-5)
    np.testing.assert_allclose(dlz.cpu().numpy(), r["d_log_z"], rtol=1e-4, atol=1e-5)
    dH, dW, AH, AW = oracle_grads(H, Wh, r["dlogits"].reshape(N * T, V))
    check_grad(dh.double().cpu().numpy().reshape(N * T, -1), dH, AH, V, "dhidden")
    check_grad(dw.double().cpu().numpy(), dW, AW, N * T, "dweight")


def test_lmhead_tbap_bwd_parity():
    w = W("pythia", B=2, K=4, T=32, V=2000, d=128, len_lo=4, len_hi=32)
    dev, gi, H, Wh = inputs(w, 13, "lattice")
    N, T, V = w.N, w.T, w.V
    gen_h = syn.gen_logp(w, 13)
    gen = torch.from_numpy(gen_h).cuda()
    n_tok = float(gi["mask"].sum())
    # IS mode "none": the clip decisions are covered by test_gpu_tbap.py; this test checks the
    # chain rule through the head with the per-token coefficients
    o, ws = tba.lmhead_tbap_fwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], gen, dev["ref_logp"],
                                dev["log_reward"], w.beta, w.K, is_mode="none", n_tok_global=n_tok,
                                check_status=True)
    dh, dw = tba.lmhead_tbap_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.coef, n_tok,
                                 chunk_rows=128)
    torch.cuda.synchronize()
    z = O.lmhead_logits(H, Wh).reshape(N, T, V)
    r = O.tbap_head(z, gi["tokens"], gi["mask"], gen_h, gi["ref_logp"], gi["log_reward"], w.beta, w.K, "none",
                    n_tok_global=n_tok)
    dH, dW, AH, AW = oracle_grads(H, Wh, r["dlogits"].reshape(N * T, V))
    check_grad(dh.double().cpu().numpy().reshape(N * T, -1), dH, AH, V, "dhidden")
    check_grad(dw.double().cpu().numpy(), dW, AW, 128, "dweight")


def test_lmhead_tb_loss_autograd_matches_raw_calls():
    w = W("toy", B=2, K=4, T=16, V=1000, d=128)
    dev, gi, H, Wh = inputs(w, 14, "normal")
    h = dev["hidden"].clone().requires_grad_(True)
    wt = dev["weight"].clone().requires_grad_(True)
    loss = tba.lmhead_tb_loss(h, wt, dev["tokens"], dev["mask"], dev["ref_logp"], dev["log_reward"], w.beta, w.K)
    loss.backward()
    o, ws = tba.lmhead_vargrad_fwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], dev["ref_logp"],
                                   dev["log_reward"], w.beta, w.K, w.N)
    dh, dw = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o.resid,
                                    2.0 / w.N)
    torch.cuda.synchronize()
    assert loss.item() == o.partial[0].item()
    assert torch.equal(h.grad, dh.to(torch.bfloat16)) and torch.equal(wt.grad, dw.to(torch.bfloat16))


def test_lmhead_bwd_qwen_dims_sampled():
    """Qwen2.5-7B dims (d = 3584, V = 152064), 128 rows: dhidden in full, dW on sampled vocab rows
    (incl. every sampled token and the last, partial, vocabulary tile)."""
    w = W("qwen", B=1, K=2, T=64)
    seed = 15
    gi = syn.group_inputs(w, seed, 0, w.B)
    N, T, d, V = w.N, w.T, w.d, w.V
    hb = torch.empty((N, T, d), dtype=torch.bfloat16, device="cuda")
    wb = torch.empty((V, d), dtype=torch.bfloat16, device="cuda")
    syn.fill_bf16_cuda(hb.view(N * T, d), seed, "hidden", 0, "normal")
    syn.fill_bf16_cuda(wb, seed, "weight", 0, "normal")
    tok, mask = torch.from_numpy(gi["tokens"]).cuda(), torch.from_numpy(gi["mask"]).cuda()
    o, ws = tba.lmhead_vargrad_fwd(hb, wb, tok, mask, torch.from_numpy(gi["ref_logp"]).cuda(),
                                   torch.from_numpy(gi["log_reward"]).cuda(), w.beta, w.K, N, check_status=True)
    dh, dw = tba.lmhead_vargrad_bwd(hb, wb, tok, mask, ws, o.resid, 2.0 / N)
    torch.cuda.synchronize()
    H = syn.bf16_bits_to_f64(syn.hidden_rows(seed, d, np.arange(N * T), "normal"))
    step = 8192
    z = np.concatenate([O.lmhead_logits(H, syn.bf16_bits_to_f64(syn.weight_rows(seed, d, np.arange(v0, min(V, v0 + step)),
                                                                                "normal")))
                        for v0 in range(0, V, step)], axis=1)
    r = O.vargrad_head(z.reshape(N, T, V), gi["tokens"], gi["mask"], gi["ref_logp"], gi["log_reward"], w.beta, w.K)
    dz = r["dlogits"].reshape(N * T, V)
    del z
    dH = np.zeros((N * T, d))
    AH = np.zeros((N * T, d))
    for v0 in range(0, V, step):
        Wc = syn.bf16_bits_to_f64(syn.weight_rows(seed, d, np.arange(v0, min(V, v0 + step)), "normal"))
        dH += dz[:, v0:v0 + step] @ Wc
        AH += np.abs(dz[:, v0:v0 + step]) @ np.abs(Wc)
    check_grad(dh.double().cpu().numpy().reshape(N * T, d), dH, AH, V, "dhidden")
    rng = np.random.default_rng(0)
    vs = np.unique(np.concatenate([gi["tokens"][gi["mask"] == 1], rng.integers(0, V, 64), np.arange(V - 40, V)]))
    dW = dz[:, vs].T @ H
    AW = np.abs(dz[:, vs]).T @ np.abs(H)
    check_grad(dw[torch.from_numpy(vs).cuda()].double().cpu().numpy(), dW, AW, N * T, "dweight")


FB_CASES = [
    ("pythia_chunks_of_1", W("pythia", B=3, K=4, T=53, V=5000, d=128), "normal", 1, 1.0, False),
    ("ragged_temp_learned_z", W("rhomath", B=2, K=4, T=96, V=3000, d=64, len_lo=0, len_hi=96), "lattice", 1,
     1 / 0.7, True),
    ("gpt2_one_chunk", W("redteam", B=4, K=2, T=20, d=96), "normal", 0, 1.0, False),
]


@pytest.mark.parametrize("name,w,kind,gpc,inv_temp,learned", FB_CASES, ids=[c[0] for c in FB_CASES])
def test_lmhead_fwd_bwd_one_call(name, w, kind, gpc, inv_temp, learned):
    """tba_lmhead_tb_loss_fwd_bwd: forward outputs and dhidden bitwise equal to the two calls (same
    tensor-core logits, same fixed-order reductions); dweight (summed over different row chunks)
    within the oracle bound."""
    dev, gi, H, Wh = inputs(w, 16, kind)
    N, T, V = w.N, w.T, w.V
    lz = torch.linspace(-1, 1, w.B, dtype=torch.float64, device="cuda") if learned else None
    args = (dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], dev["ref_logp"], dev["log_reward"], w.beta, w.K,
            N)
    r1 = tba.lmhead_vargrad_fwd_bwd(*args, inv_temp=inv_temp, log_z_param=lz, groups_per_chunk=gpc,
                                    check_status=True)
    o2, ws = tba.lmhead_vargrad_fwd(*args, inv_temp=inv_temp, log_z_param=lz, check_status=True)
    r2 = tba.lmhead_vargrad_bwd(dev["hidden"], dev["weight"], dev["tokens"], dev["mask"], ws, o2.resid, 2.0 / N,
                                inv_temp=inv_temp, log_z_param=lz, K=w.K)
    torch.cuda.synchronize()
    o1, dh1, dw1 = r1[:3]
    for f in ("seq_logp", "n_tokens", "log_z", "resid", "partial"):
        assert torch.equal(getattr(o1, f), getattr(o2, f)), f
    assert torch.equal(dh1, r2[0])
    if learned:
        assert torch.equal(r1[3], r2[2])
    z = O.lmhead_logits(H, Wh).reshape(N, T, V)
    r = O.vargrad_head(z, gi["tokens"], gi["mask"], gi["ref_logp"], gi["log_reward"], w.beta, w.K,
                       inv_temp=inv_temp, log_z=None if lz is None else lz.cpu().numpy())
    assert abs(o1.partial[0].item() - r["loss"]) <= max(1e-4 * abs(r["loss"]), 1e-5)
    dH, dW, AH, AW = oracle_grads(H, Wh, r["dlogits"].reshape(N * T, V))
    check_grad(dh1.double().cpu().numpy().reshape(N * T, -1), dH, AH, V, "dhidden")
    check_grad(dw1.double().cpu().numpy(), dW, AW, N * T, "dweight")


_PAIR_SCRIPT = r"""
import sys, torch, dataclasses
sys.path.insert(0, sys.argv[1])
import paper_2503_18929_b200 as tba, tba_synth as syn
w = dataclasses.replace(syn.WORKLOADS["pythia"], B=2, K=4, T=50, V=3000, d=320, len_lo=5, len_hi=50)
gi = syn.group_inputs(w, 17, 0, w.B)
h = torch.empty((w.N, w.T, w.d), dtype=torch.bfloat16, device="cuda")
wt = torch.empty((w.V, w.d), dtype=torch.bfloat16, device="cuda")
syn.fill_bf16_cuda(h.view(-1, w.d), 17, "hidden", 0)
syn.fill_bf16_cuda(wt, 17, "weight", 0)
dev = [torch.from_numpy(gi[k]).cuda() for k in ("tokens", "mask", "ref_logp", "log_reward")]
o, dh, dw = tba.lmhead_vargrad_fwd_bwd(h, wt, *dev, w.beta, w.K, w.N, groups_per_chunk=1)
f, _ = tba.lmhead_vargrad_fwd(h, wt, *dev, w.beta, w.K, w.N)
torch.save({"dh": dh.cpu(), "dw": dw.cpu(), "ell": f.seq_logp.cpu(), "resid": o.resid.cpu(),
            "loss": o.partial.cpu()}, sys.argv[2])
"""


def test_lmhead_bwd_pair_kernel_bitwise(tmp_path):
    """Every backward GEMM kernel gives bitwise the single-SM results (each gradient element is one
    K-ordered fp32 accumulation whatever the tile shape): the pair kernel (TBA_LMB_2SM=3) with 256 x 256
    or 256 x 512 tiles (TBA_LMB_NT2=3), K-major or MN-major dW (TBA_LMB_DW_MN)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    # (TBA_LMB_DW_MN, TBA_LMB_2SM, TBA_LMB_NT2): single-SM everywhere first
    for cfg in (("0", "0", "0"), ("0", "3", "0"), ("0", "3", "3"), ("1", "3", "3"), ("1", "3", "0")):
        f = tmp_path / f"r{''.join(cfg)}.pt"
        env = dict(os.environ, TBA_LMB_DW_MN=cfg[0], TBA_LMB_2SM=cfg[1], TBA_LMB_NT2=cfg[2], TBA_LMB_KSPLIT="1")
        subprocess.run([sys.executable, "-c", _PAIR_SCRIPT, root, str(f)], env=env, check=True, timeout=300)
        out[cfg] = torch.load(f)
    base = out[("0", "0", "0")]
    for cfg, r in out.items():
        for k in base:
            assert torch.equal(base[k], r[k]), (cfg, k)


def test_lmhead_bwd_dh_split_k(tmp_path):
    """dH = dZ W split along K (= V) into 2-4 slices on the pair kernel (TBA_LMB_KSPLIT): each slice is
    one K-ordered fp32 accumulation and the slices are summed in slice order, so everything but dH is
    bitwise the unsplit result, and dH differs only by fp32 reassociation (well inside R21's bound)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for ks in ("1", "2", "3", "4"):
        f = tmp_path / f"k{ks}.pt"
        env = dict(os.environ, TBA_LMB_2SM="3", TBA_LMB_NT2="3", TBA_LMB_KSPLIT=ks)
        subprocess.run([sys.executable, "-c", _PAIR_SCRIPT, root, str(f)], env=env, check=True, timeout=300)
        out[ks] = torch.load(f)
    base = out["1"]
    scale = base["dh"].float().abs().max().item()
    for ks, r in out.items():
        for k in base:
            if k == "dh":
                err = (r[k].float() - base[k].float()).abs().max().item()
                assert err <= 2 ** -7 * scale, (ks, err, scale)   # a bf16 rounding step at most
            else:
                assert torch.equal(base[k], r[k]), (ks, k)
