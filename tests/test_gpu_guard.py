"""Out-of-bounds guards for the row kernels' outputs (compute-sanitizer is closed on the GPU pool, so
these tests are the bounds check): the gradient writer (two-call, bf16 / fp32), the deferred-scale
pass (short and long rows, odd V) and the fused schedule write their outputs into a strided view of a
larger buffer filled with a sentinel bit pattern — guard rows before and after, pad columns after
every row, rows that start at every 2-byte offset — and every byte outside the view must still hold
the sentinel afterwards; inside the view nothing may be left unwritten (masked rows are zero-filled)."""
import dataclasses

import numpy as np
import pytest

import tba_synth as syn

from . import _harness as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2503_18929_b200 as tba  # noqa: E402

SENT16 = 0x7FA5   # a NaN bf16 pattern no kernel writes
SENT32 = 0x7FA5A5A5


def _guarded(shape, dtype, pad, guard_rows=3):
    """A [N, T, V] view with row stride V + pad inside a buffer with guard rows, filled with SENT."""
    N, T, V = shape
    rs = V + pad
    n = (N * T + 2 * guard_rows) * rs
    it = torch.int16 if dtype == torch.bfloat16 else torch.int32
    raw = torch.full((n,), SENT16 if it == torch.int16 else SENT32, dtype=it, device="cuda")
    buf = raw.view(dtype)
    view = buf[guard_rows * rs: guard_rows * rs + N * T * rs].view(N, T, rs)[:, :, :V]
    inside = torch.zeros(n, dtype=torch.bool, device="cuda")
    inside.view(-1)[guard_rows * rs: guard_rows * rs + N * T * rs].view(N * T, rs)[:, :V] = True
    return raw, view, inside


def _check(raw, inside, what):
    s = SENT16 if raw.dtype == torch.int16 else SENT32
    out = raw[~inside]
    bad = (out != s).nonzero()
    assert bad.numel() == 0, f"{what}: {bad.numel()} elements written outside the output view"
    ins = raw[inside]
    left = (ins == s).nonzero()
    assert left.numel() == 0, f"{what}: {left.numel()} output elements never written"


CASES = [
    ("redteam_odd", dataclasses.replace(syn.WORKLOADS["redteam"], B=2, K=4, T=5, len_lo=1, len_hi=5)),
    ("long_odd", dataclasses.replace(syn.WORKLOADS["redteam"], B=2, K=4, T=3, V=80001, len_lo=1, len_hi=3)),
    ("long_even", dataclasses.replace(syn.WORKLOADS["qwen"], B=1, K=4, T=3)),
    ("fp32_long", dataclasses.replace(syn.WORKLOADS["pythia"], B=1, K=4, T=3, dtype="fp32")),
    ("tiny_v", dataclasses.replace(syn.WORKLOADS["toy"], B=2, K=4, T=3, V=7)),
]


@pytest.mark.parametrize("name,w", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("pad", [0, 1, 13])
@pytest.mark.parametrize("out", ["bf16", "fp32"])
def test_outputs_stay_in_bounds(name, w, pad, out):
    inp = H.device_inputs(w, 3)
    odt = torch.bfloat16 if out == "bf16" else torch.float32
    shape = (w.N, w.T, w.V)
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, w.N)
    raw, view, inside = _guarded(shape, odt, pad)
    tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N, dlogits=view)
    torch.cuda.synchronize()
    _check(raw, inside, f"{name} two-call dlogits")
    ref = view.clone()
    raw, view, inside = _guarded(shape, odt, pad)
    tba.vargrad_fwd_deferred(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                             w.K, float(w.N), grad_unscaled=view, check_status=True)
    torch.cuda.synchronize()
    _check(raw, inside, f"{name} deferred G")
    # the same rows: G times the row coefficient is the two-call gradient (to rounding)
    c = (2.0 * o.resid / w.N).view(-1, 1, 1).to(torch.float64)
    d = (view.double() * c - ref.double()).abs()
    tol = 4 * 2.0 ** -8 * ref.double().abs() + 1e-30 + (2.0 ** -126)
    assert bool((d <= tol + 2e-6 * c.abs().clamp(min=1)).all()), f"{name}: deferred G * c differs from dlogits"
    raw, view, inside = _guarded(shape, odt, pad)
    tba.vargrad_fused(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                      float(w.N), dlogits=view)
    torch.cuda.synchronize()
    _check(raw, inside, f"{name} fused dlogits")
