"""The group-chunked two-stream schedule (tba_tb_loss_pipelined) reproduces the two-call path
bit for bit: every row, head and the final fixed-order reduction run the same arithmetic; only
the launch order differs (forward of chunk c beside the gradient writer of chunk c-1)."""
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


def _bits(t):
    return t.view(torch.int16) if t.dtype == torch.bfloat16 else t


def _two_call(inp, w, inv_temp=1.0, lz=None, dl_dtype=None):
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, w.N, inv_temp=inv_temp, log_z_param=lz)
    r = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N, inv_temp=inv_temp,
                        log_z_param=lz, K=w.K, dlogits_dtype=dl_dtype)
    d, dz = (r, None) if lz is None else r
    return o, d, dz


CASES = [
    ("toy", W("toy"), 1),
    ("rt_ragged_unaligned_gpc1", W("redteam", B=7, K=4, T=9, len_lo=0, len_hi=9), 1),
    ("rt_ragged_unaligned_gpc3", W("redteam", B=7, K=4, T=9, len_lo=0, len_hi=9), 3),  # ragged last chunk
    ("pythia_full_auto", syn.WORKLOADS["pythia"], 0),
    ("pythia_full_gpc2", syn.WORKLOADS["pythia"], 2),
    ("rhomath_small_ragged", W("rhomath", B=5, K=4, T=40, len_lo=3, len_hi=40), 2),
    ("qwen_small", W("qwen", B=3, K=4, T=8), 1),
    ("one_chunk", W("pythia", B=4, K=4, T=5), 64),
]


@pytest.mark.parametrize("name,w,gpc", CASES, ids=[c[0] for c in CASES])
def test_pipelined_equals_two_call(name, w, gpc):
    inp = H.device_inputs(w, 7)
    a, da, _ = _two_call(inp, w)
    b, _, db, _ = tba.vargrad_pipelined(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                        inp["log_reward"], w.beta, w.K, float(w.N), groups_per_chunk=gpc,
                                        check_status=True)
    torch.cuda.synchronize()
    for f in ("seq_logp", "n_tokens", "log_z", "resid", "partial"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    assert torch.equal(_bits(da), _bits(db))


def test_pipelined_single_stream_and_alias_and_fp32_out():
    w = W("pythia", B=5, K=4, T=6, V=5003)
    inp = H.device_inputs(w, 11)
    a, da, _ = _two_call(inp, w, dl_dtype=torch.float32)
    b, _, db, _ = tba.vargrad_pipelined(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                        inp["log_reward"], w.beta, w.K, float(w.N), groups_per_chunk=2,
                                        dlogits_dtype=torch.float32, aux_stream=False)
    torch.cuda.synchronize()
    assert torch.equal(a.partial, b.partial) and torch.equal(da, db)
    # dlogits aliasing logits element-for-element (in-place gradient)
    _, d2, _ = _two_call(inp, w)
    lg = inp["logits"].clone()
    c, _, dc, _ = tba.vargrad_pipelined(lg, inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                                        w.K, float(w.N), groups_per_chunk=1, dlogits=lg)
    torch.cuda.synchronize()
    assert dc.data_ptr() == lg.data_ptr()
    assert torch.equal(c.partial, a.partial) and torch.equal(_bits(lg), _bits(d2))


def test_pipelined_learned_logz_and_temperature_match_oracle():
    w = W("redteam", B=4, K=4, T=5, V=3001, len_lo=0, len_hi=5)
    inp = H.device_inputs(w, 13)
    lz = torch.linspace(-1.0, 2.0, w.B, dtype=torch.float64, device="cuda")
    a, da, dza = _two_call(inp, w, inv_temp=1.0 / 0.7, lz=lz)
    b, _, db, dzb = tba.vargrad_pipelined(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                          inp["log_reward"], w.beta, w.K, float(w.N), inv_temp=1.0 / 0.7,
                                          log_z_param=lz, groups_per_chunk=1)
    torch.cuda.synchronize()
    assert torch.equal(a.partial, b.partial) and torch.equal(a.log_z, b.log_z) and torch.equal(dza, dzb)
    assert torch.equal(_bits(da), _bits(db))
    h = inp["host"]
    ref = O.vargrad_head(H.host_logits(w, 13, 0, w.B), h["tokens"], h["mask"], h["ref_logp"], h["log_reward"],
                         w.beta, w.K, inv_temp=1.0 / 0.7, log_z=lz.cpu().numpy())
    H.assert_seq_close([b.partial[0].item()], [ref["loss"]], "loss")


def test_pipelined_in_cuda_graph_and_loss_and_grad_api():
    w = W("pythia", B=6, K=4, T=4, V=2048)
    inp = H.device_inputs(w, 17)
    a, da, _ = _two_call(inp, w)
    out = tba.ops._Fwd(w.N, w.K, torch.device("cuda"))
    ws = torch.empty(tba.workspace_bytes(w.N, w.T), dtype=torch.uint8, device="cuda")
    dl = torch.empty_like(inp["logits"])

    def run():
        tba.vargrad_pipelined(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                              w.K, float(w.N), workspace=ws, out=out, dlogits=dl, groups_per_chunk=2,
                              check_status=False)

    g = tba.CapturedStep(run)
    dl.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.partial, a.partial) and torch.equal(_bits(dl), _bits(da))
    loss, d = tba.vargrad_tb_loss_and_grad(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                           inp["log_reward"], w.beta, w.K, schedule="pipelined")
    torch.cuda.synchronize()
    assert loss.item() == a.partial[0].item() and torch.equal(_bits(d), _bits(da))


def test_pipelined_host_validation():
    w = W("toy", B=2, K=4, T=3)
    inp = H.device_inputs(w, 1)
    with pytest.raises(tba.TbaError):
        tba.vargrad_pipelined(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], -1.0,
                              w.K, float(w.N))
    with pytest.raises(tba.TbaError):
        tba.vargrad_pipelined(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                              w.K, float(w.N) - 1.0)
    # zero groups: zero partials
    w0 = W("toy", B=0, K=4, T=3)
    i0 = H.device_inputs(w0, 0)
    o0, _, _, _ = tba.vargrad_pipelined(i0["logits"], i0["tokens"], i0["mask"], i0["ref_logp"], i0["log_reward"],
                                        w.beta, w.K, 8.0)
    assert o0.partial.cpu().tolist() == [0.0, 0.0, 0.0]
