"""Randomised parity sweep (GPU vs the fp64 oracle, every element): 40 configurations drawn from a
fixed seed — vocabulary 1 .. 70 000 (aligned and odd), 0 .. 9 positions, K = 2 .. 6, padded row
strides (NaN padding), bf16 / fp32 logits and dlogits, random masks with empty responses, a
temperature, grad_out != 1, and the normaliser of a larger batch — through the TB loss
(tba_tb_loss_fwd / _bwd) and, for a quarter of them, TBA' (tba_tbap_loss_fwd / _bwd)."""
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


def _config(i):
    rng = np.random.default_rng(1000 + i)
    V = int(rng.choice([1, 2, 3, 7, 100, 1000, 4093, 8192, 32000, 50257, 69997]))
    T = int(rng.integers(0, 10))
    K = int(rng.integers(2, 7))
    B = int(rng.integers(1, 4))
    dtype = "fp32" if rng.random() < 0.3 else "bf16"
    out = "fp32" if rng.random() < 0.3 else dtype
    pad = int(rng.choice([0, 0, 8, 37]))
    inv_temp = float(rng.choice([1.0, 1.0, 1.0 / 0.7, 2.0]))
    grad_out = float(rng.choice([1.0, -0.5, 3.0]))
    n_global = B * K * int(rng.choice([1, 1, 4]))
    tbap = rng.random() < 0.25
    return rng, dict(V=V, T=T, K=K, B=B, dtype=dtype, out=out, pad=pad, inv_temp=inv_temp, grad_out=grad_out,
                     n_global=n_global, tbap=tbap)


@pytest.mark.parametrize("i", range(40))
def test_random_configuration(i):
    rng, c = _config(i)
    V, T, K, B = c["V"], c["T"], c["K"], c["B"]
    N = B * K
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    odt = torch.bfloat16 if c["out"] == "bf16" else torch.float32
    z = rng.normal(0.0, 2.5, (N, T, V))
    if V > 1 and T > 0:
        tokens = rng.integers(0, V, (N, T))
        hot = rng.random((N, T)) < 0.3                     # some confident tokens
        z[np.arange(N)[:, None], np.arange(T)[None, :], tokens] += np.where(hot, 18.0, 0.0)
    else:
        tokens = np.zeros((N, T), np.int64)
    z = syn.bf16_bits_to_f64(syn.f32_to_bf16_bits(z.astype(np.float32))) if c["dtype"] == "bf16" else \
        z.astype(np.float32).astype(np.float64)
    mask = (rng.random((N, T)) < 0.75).astype(np.uint8)
    if N > 1 and T > 0:
        mask[1] = 0                                         # an empty response
    tokens = np.where(mask == 1, tokens, -1).astype(np.int64)
    ref = rng.normal(-3.0 * T, 2.0, N).astype(np.float32).astype(np.float64)
    rew = rng.normal(0.0, 1.0, N).astype(np.float32).astype(np.float64)
    beta = float(rng.choice([1.0, 0.05, 0.3]))
    rs = V + c["pad"]
    buf = torch.full((N, T, rs), float("nan"), dtype=tdt, device="cuda")
    buf[:, :, :V] = torch.from_numpy(z).to(tdt)
    lg = buf[:, :, :V]
    tk, mk = torch.from_numpy(tokens).cuda(), torch.from_numpy(mask).cuda()
    rf, rw = torch.from_numpy(ref).cuda(), torch.from_numpy(rew).cuda()
    go = torch.tensor(c["grad_out"], dtype=torch.float64, device="cuda")
    what = f"cfg {i} {c}"
    if c["tbap"]:
        gen = (rng.normal(-1.0, 1.0, (N, T)) * mask).astype(np.float32)
        ntok = max(int(mask.sum()), 1)
        o, ws = tba.tbap_fwd(lg, tk, mk, torch.from_numpy(gen).cuda(), rf, rw, beta, K, "clip", 0.0, 8.0, float(ntok),
                             check_status=True)
        d = tba.tbap_bwd(lg, tk, mk, ws, o.coef, float(ntok), grad_out=go, dlogits_dtype=odt)
        torch.cuda.synchronize()
        r = O.tbap_head(z, tokens, mask, gen, ref, rew, beta, K, "clip", 0.0, 8.0, ntok, grad_out=c["grad_out"])
        H.assert_seq_close(o.seq_logp.cpu().numpy(), r["ell"], f"{what} seq_logp")
        H.assert_seq_close([o.partial[0].item()], [r["loss"]], f"{what} loss")
        scale = -r["coef"] / ntok * c["grad_out"]
    else:
        o, ws = tba.vargrad_fwd(lg, tk, mk, rf, rw, beta, K, float(c["n_global"]), check_status=True,
                                inv_temp=c["inv_temp"])
        d = tba.vargrad_bwd(lg, tk, mk, ws, o.resid, 2.0 / c["n_global"], grad_out=go, dlogits_dtype=odt,
                            inv_temp=c["inv_temp"])
        torch.cuda.synchronize()
        r = O.vargrad_head(z, tokens, mask, ref, rew, beta, K, n_global=c["n_global"], grad_out=c["grad_out"],
                           inv_temp=c["inv_temp"])
        H.assert_seq_close(o.seq_logp.cpu().numpy(), r["ell"], f"{what} seq_logp")
        tz, te = H.seq_tols(r["ell"], K)
        H.assert_close_tol(o.resid.cpu().numpy(), r["eps"], te, f"{what} resid")
        H.assert_seq_close([o.partial[0].item()], [r["loss"]], f"{what} loss")
        scale = np.repeat((2.0 * r["eps"] / c["n_global"] * c["grad_out"] * c["inv_temp"])[:, None], T, axis=1)
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), mask.sum(1))
    dd = d.double().cpu().numpy()
    for s in range(N):
        for t in range(T):
            H.assert_dlogits_close(dd[s, t], r["dlogits"][s, t], float(scale[s, t]), c["out"], f"{what} s={s} t={t}")
