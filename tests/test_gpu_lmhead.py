"""GPU parity of the LM-head-fused head (NEXT 3; tba_lmhead_seq_logprob / tba_lmhead_tb_loss_fwd)
against the fp64 oracle z = W h -> log-softmax (oracle/tba_oracle.py, pinned in
tests/test_oracle_lmhead.py).

Tolerances: on "lattice" inputs (entries in {-2..2}/4) every partial sum of
every dot product is exact in fp32, so the logits are exact whatever the tensor cores'
accumulation order and only the softmax epilogue's error remains: |d lp| <= 1e-6 per token.
On "normal" inputs the fp32 accumulation of the d-term dot products adds, per token,
|d lp| <= 4 sqrt(d) 2^-24 (A_y + max_v A_v) + 1e-6 with A_v = sum_i |h_i| |W_vi| (the
statistical sqrt(d) growth of independent rounding errors, 4 standard deviations)."""
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


def lm_inputs(w, seed, kind="normal", pad_h=0, pad_w=0):
    gi = syn.group_inputs(w, seed, 0, w.B)
    N, T, d, V = w.N, w.T, w.d, w.V
    hb = torch.full((N, T, d + pad_h), float("nan"), dtype=torch.bfloat16, device="cuda")
    wb = torch.full((V, d + pad_w), float("nan"), dtype=torch.bfloat16, device="cuda")
    if N * T:
        syn.fill_bf16_cuda(hb.view(N * T, d + pad_h)[:, :d], seed, "hidden", 0, kind)
    syn.fill_bf16_cuda(wb[:, :d], seed, "weight", 0, kind)
    return dict(hidden=hb[:, :, :d], weight=wb[:, :d], tokens=torch.from_numpy(gi["tokens"]).cuda(),
                mask=torch.from_numpy(gi["mask"]).cuda(), ref_logp=torch.from_numpy(gi["ref_logp"]).cuda(),
                log_reward=torch.from_numpy(gi["log_reward"]).cuda(), host=gi)


def oracle_rows(w, seed, rows, toks, kind, inv_temp=1.0, chunk=8192):
    """Oracle log-probs of the given global rows and their tolerance (module docstring)."""
    h = syn.bf16_bits_to_f64(syn.hidden_rows(seed, w.d, rows, kind))
    habs = np.abs(h)
    zs, amax = [], np.zeros(len(rows))
    ay = np.zeros(len(rows))
    for v0 in range(0, w.V, chunk):
        v1 = min(w.V, v0 + chunk)
        wv = syn.bf16_bits_to_f64(syn.weight_rows(seed, w.d, np.arange(v0, v1), kind))
        zs.append(O.lmhead_logits(h, wv))
        a = habs @ np.abs(wv).T
        amax = np.maximum(amax, a.max(1))
        sel = (toks >= v0) & (toks < v1)
        ay[sel] = a[np.flatnonzero(sel), toks[sel] - v0]
    z = np.concatenate(zs, axis=1) * inv_temp
    lp = np.array([O.token_logprob(z[r], int(toks[r]))[0] for r in range(len(rows))])
    if kind == "lattice":
        tol = np.full(len(rows), 1e-6) + 1e-8 * np.abs(lp)
    else:
        tol = 4 * math.sqrt(w.d) * 2.0 ** -24 * inv_temp * (ay + amax) + 1e-6
    return lp, tol


def check_seq(w, seed, kind, got_ell, got_ntok, inv_temp=1.0):
    tok, mask = syn.tokens_and_mask(w, seed)
    N, T = tok.shape
    valid = np.flatnonzero(mask.reshape(-1))
    lp = np.zeros(N * T)
    tol = np.zeros(N * T)
    if len(valid):
        lp[valid], tol[valid] = oracle_rows(w, seed, valid, tok.reshape(-1)[valid], kind, inv_temp)
    ell = np.array([math.fsum(lp.reshape(N, T)[s]) for s in range(N)])
    tol_s = tol.reshape(N, T).sum(1)
    np.testing.assert_array_equal(got_ntok, mask.sum(1))
    err = np.abs(np.asarray(got_ell) - ell)
    assert np.all(err <= tol_s), f"seq_logp off: err {err[:8]} tol {tol_s[:8]}"
    return ell, err


LATTICE = [
    ("tiny", W("toy", B=1, K=1, T=1, V=256, d=64)),
    ("ragged_tails", W("toy", B=3, K=1, T=100, V=1000, d=200, len_lo=0, len_hi=100)),
    ("gpt2_dims", W("redteam", B=2, K=1, T=77, len_lo=1, len_hi=77)),
    ("four_row_blocks", W("pythia", B=2, K=4, T=64, V=5000, d=128)),
    # responses <= 128 of T = 256: every second row block is fully masked and skipped
    ("skipped_row_blocks", W("rhomath", B=1, K=4, T=256, V=700, d=64, len_lo=0, len_hi=128)),
]


@pytest.mark.parametrize("name,w", LATTICE, ids=[c[0] for c in LATTICE])
def test_lmhead_lattice_exact_logits(name, w):
    inp = lm_inputs(w, 3, "lattice", pad_h=8, pad_w=16)
    ell, nt = tba.lmhead_seq_logprob(inp["hidden"], inp["weight"], inp["tokens"], inp["mask"], check_status=True)
    torch.cuda.synchronize()
    check_seq(w, 3, "lattice", ell.cpu().numpy(), nt.cpu().numpy())


def test_lmhead_normal_qwen_dims_one_row_block():
    w = W("qwen", B=2, K=1, T=64)
    inp = lm_inputs(w, 5, "normal")
    ell, nt = tba.lmhead_seq_logprob(inp["hidden"], inp["weight"], inp["tokens"], inp["mask"], check_status=True)
    torch.cuda.synchronize()
    check_seq(w, 5, "normal", ell.cpu().numpy(), nt.cpu().numpy())


def test_lmhead_tb_head_temperature_and_learned_logz():
    w = W("pythia", B=3, K=4, T=9, V=3001, d=96, len_lo=0, len_hi=9)
    inp = lm_inputs(w, 7, "lattice")
    h = inp["host"]
    rows = np.arange(w.N * w.T)
    hid = syn.bf16_bits_to_f64(syn.hidden_rows(7, w.d, rows, "lattice"))
    wt = syn.bf16_bits_to_f64(syn.weight_rows(7, w.d, np.arange(w.V), "lattice"))
    logits = O.lmhead_logits(hid, wt).reshape(w.N, w.T, w.V)
    for inv_temp, lz in ((1.0, None), (1 / 0.7, np.linspace(-1, 2, w.B))):
        lzt = None if lz is None else torch.from_numpy(lz).cuda()
        o, _ = tba.lmhead_vargrad_fwd(inp["hidden"], inp["weight"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                      inp["log_reward"], w.beta, w.K, float(w.N), inv_temp=inv_temp,
                                      log_z_param=lzt, check_status=True)
        torch.cuda.synchronize()
        ref = O.vargrad_head(logits, h["tokens"], h["mask"], h["ref_logp"], h["log_reward"], w.beta, w.K,
                             inv_temp=inv_temp, log_z=lz, want_grad=False)
        tol = 1e-6 * (1 + h["mask"].sum(1))
        assert np.all(np.abs(o.seq_logp.cpu().numpy() - ref["ell"]) <= tol)
        np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), h["mask"].sum(1))
        assert np.all(np.abs(o.resid.cpu().numpy() - ref["eps"]) <= 2 * tol.max())  # eps = log Z - delta
        assert abs(o.partial[0].item() - ref["loss"]) <= 1e-5 * max(1.0, abs(ref["loss"]))
        assert o.partial[1].item() == w.N and o.partial[2].item() == w.B


def test_lmhead_edges_and_validation():
    # an all-masked sequence gives 0 / 0; zero sequences are a no-op
    w = W("toy", B=2, K=1, T=5, V=300, d=64, len_lo=0, len_hi=5)
    inp = lm_inputs(w, 11, "lattice")
    inp["mask"][0].zero_()
    ell, nt = tba.lmhead_seq_logprob(inp["hidden"], inp["weight"], inp["tokens"], inp["mask"], check_status=True)
    assert ell[0].item() == 0.0 and nt[0].item() == 0
    w0 = W("toy", B=0, K=1, T=5, V=300, d=64)
    i0 = lm_inputs(w0, 0, "lattice")
    e0, n0 = tba.lmhead_seq_logprob(i0["hidden"], i0["weight"], i0["tokens"], i0["mask"])
    assert e0.numel() == 0
    # a token outside [0, V) at a valid position is reported
    bad = inp["tokens"].clone()
    bad[1, 0] = w.V
    with pytest.raises(ValueError, match="device status 1"):
        tba.lmhead_seq_logprob(inp["hidden"], inp["weight"], bad, inp["mask"], check_status=True)
    # d must be a multiple of 8 (16-byte TMA strides)
    hid = torch.zeros(2, 5, 12, dtype=torch.bfloat16, device="cuda")
    wt = torch.zeros(300, 12, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tba.TbaError):
        tba.lmhead_seq_logprob(hid, wt, inp["tokens"], inp["mask"])


def test_lmhead_fullsize_qwen_shard_sampled_sequence():
    """The bench configuration (Qwen shard: 65536 rows x V = 152064 x d = 3584, persistent grid
    of one CTA per SM): the first and the last sequence's log-probs against the oracle."""
    w = syn.WORKLOADS["qwen_shard"]
    N, T, d, V = w.N, w.T, w.d, w.V
    gi = syn.group_inputs(w, 1, 0, w.B)
    hid = torch.empty((N, T, d), dtype=torch.bfloat16, device="cuda")
    wt = torch.empty((V, d), dtype=torch.bfloat16, device="cuda")
    syn.fill_bf16_cuda(hid.view(N * T, d), 1, "hidden", 0)
    syn.fill_bf16_cuda(wt, 1, "weight", 0)
    tok, mask = torch.from_numpy(gi["tokens"]).cuda(), torch.from_numpy(gi["mask"]).cuda()
    ell, nt = tba.lmhead_seq_logprob(hid, wt, tok, mask, check_status=True)
    torch.cuda.synchronize()
    ell = ell.cpu().numpy()
    for s in (0, N - 1):
        rows = np.arange(s * T, (s + 1) * T)
        lp, tol = oracle_rows(w, 1, rows, gi["tokens"].reshape(-1)[rows], "normal")
        assert abs(ell[s] - math.fsum(lp)) <= tol.sum(), (s, ell[s], math.fsum(lp), tol.sum())
    assert nt.cpu().numpy().tolist() == [T] * N


@pytest.mark.parametrize("kind", ["normal", "lattice"])
def test_synth_cuda_twin_bf16(kind):
    for which, gen in (("hidden", syn.hidden_rows), ("weight", syn.weight_rows)):
        buf = torch.zeros((300, 136), dtype=torch.bfloat16, device="cuda")
        syn.fill_bf16_cuda(buf[:, :128], 9, which, 1000, kind)
        got = buf[:, :128].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        np.testing.assert_array_equal(got, gen(9, 128, np.arange(1000, 1300), kind))
        assert buf[:, 128:].abs().sum().item() == 0  # the row padding is untouched


def test_lmhead_token_logprob_and_tbap_match_oracle():
    w = W("qwen", B=2, K=4, T=7, V=4001, d=136, len_lo=2, len_hi=7, beta=0.005)
    inp = lm_inputs(w, 13, "lattice")
    h = inp["host"]
    rows = np.arange(w.N * w.T)
    hid = syn.bf16_bits_to_f64(syn.hidden_rows(13, w.d, rows, "lattice"))
    wt = syn.bf16_bits_to_f64(syn.weight_rows(13, w.d, np.arange(w.V), "lattice"))
    logits = O.lmhead_logits(hid, wt).reshape(w.N, w.T, w.V)
    # per-token log-probs (temperature 0.7)
    tl = tba.lmhead_token_logprob(inp["hidden"], inp["weight"], inp["tokens"], inp["mask"], inv_temp=1 / 0.7,
                                  check_status=True).cpu().numpy()
    for s in range(w.N):
        for t in range(w.T):
            if h["mask"][s, t]:
                ref = O.token_logprob(logits[s, t] / 0.7, int(h["tokens"][s, t]))[0]
                assert abs(tl[s, t] - ref) <= 1e-6 + 1e-8 * abs(ref), (s, t, tl[s, t], ref)
            else:
                assert tl[s, t] == 0.0
    # TBA' (Eq. 16) from hidden states vs the oracle on the same logits
    gen = syn.gen_logp(w, 13)
    ntok = int(h["mask"].sum())
    o, _ = tba.lmhead_tbap_fwd(inp["hidden"], inp["weight"], inp["tokens"], inp["mask"], torch.from_numpy(gen).cuda(),
                               inp["ref_logp"], inp["log_reward"], w.beta, w.K, "none", n_tok_global=ntok,
                               check_status=True)
    torch.cuda.synchronize()
    ref = O.tbap_head(logits, h["tokens"], h["mask"], gen, h["ref_logp"], h["log_reward"], w.beta, w.K, "none",
                      0.0, 0.0, want_grad=False)
    tol = 1e-6 * (1 + h["mask"].sum(1))
    assert np.all(np.abs(o.seq_logp.cpu().numpy() - ref["ell"]) <= tol)
    assert np.all(np.abs(o.adv.cpu().numpy() - ref["adv"]) <= 2 * w.beta * tol.max() + 1e-9)
    assert abs(o.partial[0].item() - ref["loss"]) <= 1e-5 * max(1.0, abs(ref["loss"]))
