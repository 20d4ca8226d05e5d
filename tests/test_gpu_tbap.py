"""GPU parity of the TBA' token-level rule (Eq. 16; tba_tbap_loss_fwd/bwd) against the oracle."""
import dataclasses
import math

import numpy as np
import pytest

import tba_synth as syn
from oracle import tba_oracle as O

from . import _harness as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2503_18929_b200 as tba  # noqa: E402

MODES = [("none", 0.0, 0.0), ("clip", 0.0, 8.0), ("icepop", 0.5, 2.0)]


def W(name, **kw):
    return dataclasses.replace(syn.WORKLOADS[name], **kw)


def _compare(w, seed, mode, lo, hi, grad_out=1.0, dl_dtype=None):
    inp = H.device_inputs(w, seed)
    gen = syn.gen_logp(w, seed)
    g_dev = torch.from_numpy(gen).cuda()
    ntok = int(inp["host"]["mask"].sum())
    o, ws = tba.tbap_fwd(inp["logits"], inp["tokens"], inp["mask"], g_dev, inp["ref_logp"], inp["log_reward"], w.beta,
                         w.K, mode, lo, hi, ntok, check_status=True)
    go = torch.tensor(grad_out, dtype=torch.float64, device="cuda")
    d = tba.tbap_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.coef, ntok, grad_out=go,
                     dlogits_dtype=dl_dtype)
    torch.cuda.synchronize()
    h = inp["host"]
    lg = H.host_logits(w, seed, 0, w.B)
    ref = O.tbap_head(lg, h["tokens"], h["mask"], gen, h["ref_logp"], h["log_reward"], w.beta, w.K, mode, lo, hi,
                      grad_out=grad_out)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp")
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), ref["n_tok"])
    H.assert_seq_close(o.adv.cpu().numpy(), ref["adv"], "adv")
    # coefficients: where lambda sits within 1e-5 of an IS threshold, both decisions are valid
    coef = o.coef.cpu().numpy().astype(np.float64)
    lam = np.exp(ref["lp"] - gen.astype(np.float64))
    near = np.zeros_like(lam, dtype=bool)
    for thr in ([lo, hi] if mode != "none" else []):
        if thr > 0:
            near |= np.abs(lam - thr) <= 1e-5 * thr
    ok = np.abs(coef - ref["coef"]) <= np.maximum(1e-4 * np.abs(ref["coef"]), 1e-6)
    assert np.all(ok | near), f"coef mismatch at {np.argwhere(~(ok | near))[:5]}"
    if not near.any():
        H.assert_seq_close([o.partial[0].item()], [ref["loss"]], "surrogate loss")
    dd = d.float().cpu().numpy().astype(np.float64)
    dt = "bf16" if d.dtype == torch.bfloat16 else "fp32"
    for s in range(w.N):
        for t in range(w.T):
            if near[s, t]:
                continue
            H.assert_dlogits_close(dd[s, t], ref["dlogits"][s, t], ref["coef"][s, t] / ntok * grad_out, dt,
                                   f"s={s} t={t}")
    return o, d, ref


@pytest.mark.parametrize("mode,lo,hi", MODES)
def test_tbap_qwen_vocab(mode, lo, hi):
    _compare(W("qwen", B=2, K=4, T=6), 0, mode, lo, hi)


@pytest.mark.parametrize("mode,lo,hi", MODES)
def test_tbap_ragged_unaligned(mode, lo, hi):
    _compare(W("redteam", B=2, K=3, T=7, len_lo=0, len_hi=7), 1, mode, lo, hi)


def test_tbap_fp32_logits_and_grad_out():
    _compare(W("toy", B=2, K=4, T=5), 2, "clip", 0.0, 8.0, grad_out=-1.5)


def test_tbap_beta0_fp32_dlogits():
    _compare(W("rhomath", B=2, K=4, T=5, V=4093, len_lo=1, len_hi=5, beta=0.0), 3, "icepop", 0.5, 2.0,
             dl_dtype=torch.float32)


def test_tbap_autograd_and_zero_groups():
    w = W("pythia", B=2, K=4, T=3, V=2048)
    inp = H.device_inputs(w, 5)
    gen = torch.from_numpy(syn.gen_logp(w, 5)).cuda()
    lg = inp["logits"].clone().requires_grad_(True)
    loss, aux = tba.tbap_loss(lg, inp["tokens"], inp["mask"], gen, inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                              return_aux=True)
    loss.backward()
    h = inp["host"]
    ref = O.tbap_head(H.host_logits(w, 5, 0, w.B), h["tokens"], h["mask"], gen.cpu().numpy(), h["ref_logp"],
                      h["log_reward"], w.beta, w.K)
    H.assert_seq_close([loss.item()], [ref["loss"]], "loss")
    assert lg.grad is not None and lg.grad.shape == lg.shape
    # a rank with no groups contributes zero partials
    w0 = W("pythia", B=0, K=4, T=3, V=2048)
    i0 = H.device_inputs(w0, 0)
    o0, _ = tba.tbap_fwd(i0["logits"], i0["tokens"], i0["mask"], torch.zeros((0, 3), device="cuda"),
                         i0["ref_logp"], i0["log_reward"], 0.1, 4, n_tok_global=10.0)
    assert o0.partial.cpu().tolist() == [0.0, 0.0, 0.0]


def test_tbap_on_policy_matches_scaled_tb_gradient():
    """lambda = 1, no IS: TBA' dlogits = (beta N / (2 n_tok)) x VarGrad TB dlogits (Eq. 7 <-> 16),
    both computed on the GPU (fp32 dlogits)."""
    w = W("pythia", B=2, K=4, T=4, V=3000)
    inp = H.device_inputs(w, 6)
    h = inp["host"]
    lp_host = np.zeros((w.N, w.T), np.float32)
    lg = H.host_logits(w, 6, 0, w.B)
    for s in range(w.N):
        for t in range(w.T):
            lp_host[s, t] = O.token_logprob(lg[s, t], int(h["tokens"][s, t]))[0]
    gen = torch.from_numpy(lp_host).cuda()  # on-policy up to fp32 rounding of the log-probs
    ntok = int(h["mask"].sum())
    o, ws = tba.tbap_fwd(inp["logits"], inp["tokens"], inp["mask"], gen, inp["ref_logp"], inp["log_reward"], w.beta,
                         w.K, "none", n_tok_global=ntok)
    dp = tba.tbap_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.coef, ntok, dlogits_dtype=torch.float32)
    ot, wst = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                              w.K, w.N)
    dt = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], wst, ot.resid, 2.0 / w.N,
                         dlogits_dtype=torch.float32)
    torch.cuda.synchronize()
    scale = w.beta * w.N / (2 * ntok)
    np.testing.assert_allclose(o.adv.cpu().numpy(), -w.beta * ot.resid.cpu().numpy(), rtol=1e-6, atol=1e-9)
    assert torch.allclose(dp.double(), scale * dt.double(), rtol=1e-4, atol=1e-9)


def test_tbap_deferred_scale_matches_oracle():
    """TBA' with the deferred-scale row pass: -(coef/n_tok) * G equals the oracle's dlogits."""
    w = W("qwen", B=2, K=4, T=5)
    inp = H.device_inputs(w, 8)
    gen = syn.gen_logp(w, 8)
    ntok = int(inp["host"]["mask"].sum())
    G = torch.empty(inp["logits"].shape, dtype=torch.float32, device="cuda")
    o, ws = tba.tbap_fwd(inp["logits"], inp["tokens"], inp["mask"], torch.from_numpy(gen).cuda(), inp["ref_logp"],
                         inp["log_reward"], w.beta, w.K, "clip", 0.0, 8.0, ntok, grad_unscaled=G, check_status=True)
    torch.cuda.synchronize()
    h = inp["host"]
    ref = O.tbap_head(H.host_logits(w, 8, 0, w.B), h["tokens"], h["mask"], gen, h["ref_logp"], h["log_reward"],
                      w.beta, w.K, "clip", 0.0, 8.0)
    H.assert_seq_close(o.adv.cpu().numpy(), ref["adv"], "adv")
    coef = o.coef.cpu().numpy().astype(np.float64)
    g = G.double().cpu().numpy()
    for s in range(w.N):
        for t in range(w.T):
            c = -coef[s, t] / ntok
            H.assert_dlogits_close(g[s, t] * c, ref["dlogits"][s, t], c, "fp32", f"s={s} t={t}")
