"""GPU parity of the TB head variants (learned log Z, Eq. 3; inverse temperature) vs the oracle."""
import dataclasses

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


def W(name, **kw):
    return dataclasses.replace(syn.WORKLOADS[name], **kw)


@pytest.mark.parametrize("inv_temp,learned", [(1.0, True), (1 / 0.7, False), (1 / 0.7, True), (2.0, False)])
@pytest.mark.parametrize("wl", ["pythia_small", "toy"])
def test_variants_match_oracle(inv_temp, learned, wl):
    w = W("pythia", B=2, K=4, T=5, V=5003) if wl == "pythia_small" else syn.WORKLOADS["toy"]
    inp = H.device_inputs(w, 3)
    h = inp["host"]
    lz = np.linspace(-40.0, 30.0, w.B) if learned else None
    lz_dev = torch.tensor(lz, dtype=torch.float64, device="cuda") if learned else None
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, w.N, check_status=True, inv_temp=inv_temp, log_z_param=lz_dev)
    r = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N, inv_temp=inv_temp,
                        log_z_param=lz_dev, K=w.K)
    d, dz = (r, None) if lz is None else r
    torch.cuda.synchronize()
    ref = O.vargrad_head(H.host_logits(w, 3, 0, w.B), h["tokens"], h["mask"], h["ref_logp"], h["log_reward"], w.beta,
                         w.K, inv_temp=inv_temp, log_z=lz)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp")
    H.assert_seq_close(o.log_z.cpu().numpy(), ref["log_z"], "log_z")
    H.assert_seq_close(o.resid.cpu().numpy(), ref["eps"], "resid")
    H.assert_seq_close([o.partial[0].item()], [ref["loss"]], "loss")
    if learned:
        H.assert_seq_close(dz.cpu().numpy(), ref["d_log_z"], "d_log_z")
    dd = d.float().cpu().numpy().astype(np.float64)
    dt = "bf16" if d.dtype == torch.bfloat16 else "fp32"
    for s in range(w.N):
        for t in range(w.T):
            H.assert_dlogits_close(dd[s, t], ref["dlogits"][s, t], inv_temp * 2 * ref["eps"][s] / w.N, dt)


def test_learned_log_z_autograd():
    w = W("redteam", B=3, K=4, T=4, V=3001)
    inp = H.device_inputs(w, 4)
    lz = torch.tensor([-3.0, 0.5, 12.0], dtype=torch.float64, device="cuda", requires_grad=True)
    lg = inp["logits"].clone().requires_grad_(True)
    loss = tba.vargrad_tb_loss(lg, inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                               log_z=lz)
    (2.0 * loss).backward()
    h = inp["host"]
    ref = O.vargrad_head(H.host_logits(w, 4, 0, w.B), h["tokens"], h["mask"], h["ref_logp"], h["log_reward"], w.beta,
                         w.K, log_z=lz.detach().cpu().numpy(), grad_out=2.0)
    H.assert_seq_close([loss.item()], [ref["loss"]], "loss")
    H.assert_seq_close(lz.grad.cpu().numpy(), ref["d_log_z"], "d_log_z")
    g = lg.grad.double().cpu().numpy()
    for s in range(w.N):
        for t in range(w.T):
            H.assert_dlogits_close(g[s, t], ref["dlogits"][s, t], 4 * ref["eps"][s] / w.N, "bf16")


def test_bad_temperature_rejected():
    w = W("toy", B=1)
    inp = H.device_inputs(w, 0)
    for a in (0.0, -1.0, float("nan")):
        with pytest.raises(tba.TbaError):
            tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], 1.0, 4,
                            4.0, inv_temp=a)
