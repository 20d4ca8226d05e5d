"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element,
on the same seeded inputs. Tolerances (north_star): per-sequence log-probs,
log Z, residuals and the loss to relative 1e-4 (absolute 1e-5 near zero); token counts
bit-exact; dlogits within 1 bf16 ulp (bf16) or 2e-6*max(1,|c_seq|) (fp32)."""
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


def W(name, **kw):
    return dataclasses.replace(syn.WORKLOADS[name], **kw)


def run_gpu(inp, w, n_global=None, dlogits_dtype=None, grad_out=None, check=True):
    N = inp["tokens"].shape[0]
    ng = n_global or N
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, ng, check_status=check)
    d = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / ng, grad_out=grad_out,
                        dlogits_dtype=dlogits_dtype)
    torch.cuda.synchronize()
    return o, d


def compare_full(w, seed, row_stride=None, dlogits_dtype=None, grad_out=1.0):
    inp = H.device_inputs(w, seed, row_stride=row_stride)
    go = torch.tensor(grad_out, dtype=torch.float64, device="cuda")
    o, d = run_gpu(inp, w, dlogits_dtype=dlogits_dtype, grad_out=go)
    lg = H.host_logits(w, seed, 0, w.B)
    h = inp["host"]
    ref = O.vargrad_head(lg, h["tokens"], h["mask"], h["ref_logp"], h["log_reward"], w.beta, w.K, grad_out=grad_out)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp")
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), ref["n_tok"])
    H.assert_seq_close(o.log_z.cpu().numpy(), ref["log_z"], "log_z")
    H.assert_seq_close(o.resid.cpu().numpy(), ref["eps"], "resid")
    p = o.partial.cpu().numpy()
    H.assert_seq_close([p[0]], [ref["loss"]], "loss")
    assert p[1] == w.N and p[2] == w.B
    dd = d.float().cpu().numpy().astype(np.float64)
    out_dt = "bf16" if d.dtype == torch.bfloat16 else "fp32"
    N = w.N
    for s in range(N):
        c = 2.0 * ref["eps"][s] / N * grad_out
        for t in range(w.T):
            H.assert_dlogits_close(dd[s, t], ref["dlogits"][s, t], c, out_dt, f"s={s} t={t}")
    return o, d, ref


# ------------------------------------------------------------------------------- generator twin
@pytest.mark.parametrize("dtype,V,rs", [("bf16", 50257, 50264), ("fp32", 1000, 1000), ("bf16", 152064, 152064)])
def test_generator_twins_bit_identical(dtype, V, rs):
    rows = 7
    buf = torch.empty((rows, rs), dtype=H.torch_dtype(dtype), device="cuda")
    syn.fill_logits_cuda(buf[:, :V], 3, 1234, V)
    if rs > V:
        assert torch.isnan(buf[:, V:].float()).all()
    host = syn.logits_rows(3, V, np.arange(1234, 1234 + rows), dtype)
    got = buf[:, :V].cpu()
    got = got.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else got.numpy()
    np.testing.assert_array_equal(got, host)


# ------------------------------------------------------------------------------- full parity, small shapes
def test_toy_full():
    compare_full(syn.WORKLOADS["toy"], 0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bf16_unaligned_cta_path(seed):
    # V = 50257 (GPT-2): odd row length, rows start at every 2-byte offset mod 16
    compare_full(W("redteam", B=2, K=3, T=5, len_lo=2, len_hi=5), seed)


def test_bf16_warp_path_ragged():
    compare_full(W("rhomath", B=3, K=4, T=9, V=4093, len_lo=0, len_hi=9), 5)


def test_fp32_cta_path_unaligned():
    compare_full(W("toy", B=2, K=2, T=3, V=20011), 4)


def test_padded_row_stride_nan_padding():
    compare_full(W("pythia", B=2, K=2, T=3, V=3000), 6, row_stride=3072)


def test_bf16_logits_fp32_dlogits_and_grad_out():
    compare_full(W("pythia", B=2, K=3, T=4, V=5003), 7, dlogits_dtype=torch.float32, grad_out=-2.5)


def test_k40_and_k2():
    compare_full(W("rhomath", B=1, K=40, T=3, V=777, len_lo=1, len_hi=3), 8)
    compare_full(W("qwen", B=3, K=2, T=4, V=1531), 9)


def test_qwen_vocab_small_T():
    compare_full(W("qwen", B=1, K=4, T=3), 0)


# ------------------------------------------------------------------------------- edge cases
def _edge_inputs(N, T, V, K, dtype=torch.bfloat16, seed=0):
    g = torch.Generator().manual_seed(seed)
    z = (torch.randn(N, T, V, generator=g) * 2).to(dtype)
    tok = torch.randint(0, V, (N, T), generator=g)
    mask = torch.ones(N, T, dtype=torch.uint8)
    ref = torch.randn(N, generator=g, dtype=torch.float64) * 3 - 10
    rew = torch.rand(N, generator=g, dtype=torch.float64)
    return z, tok, mask, ref, rew


def _oracle_compare(z, tok, mask, ref, rew, beta, K, dl_dtype=None):
    dev = dict(logits=z.cuda(), tokens=tok.cuda(), mask=mask.cuda(), ref_logp=ref.cuda(), log_reward=rew.cuda())
    w = dataclasses.replace(syn.WORKLOADS["toy"], beta=beta, K=K)
    o, d = run_gpu(dev, w, dlogits_dtype=dl_dtype)
    zz = z.double().numpy()
    r = O.vargrad_head(zz, tok.numpy(), mask.numpy(), ref.numpy(), rew.numpy(), beta, K)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), r["ell"], "seq_logp")
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), r["n_tok"])
    H.assert_seq_close(o.resid.cpu().numpy(), r["eps"], "resid")
    dd = d.double().cpu().numpy()
    dt = "bf16" if d.dtype == torch.bfloat16 else "fp32"
    for s in range(z.shape[0]):
        for t in range(z.shape[1]):
            H.assert_dlogits_close(dd[s, t], r["dlogits"][s, t], 2 * r["eps"][s] / z.shape[0], dt)
    return o, d, r


def test_neg_inf_logits_and_empty_sequences():
    z, tok, mask, ref, rew = _edge_inputs(6, 4, 9000, 3)
    z[0, 0, :4096] = float("-inf")       # a fully -inf first tile
    z[1, 2, ::3] = float("-inf")
    tok[1, 2] = 3 * (int(tok[1, 2]) // 3) + 1   # the sampled token itself stays finite
    tok[0, 0] = 5000
    mask[2] = 0                          # empty response (legal: ell = 0, n_tok = 0)
    mask[4, 2:] = 0
    tok[mask == 0] = -7                  # garbage where masked
    _oracle_compare(z, tok, mask, ref, rew, 0.3, 3)


@pytest.mark.parametrize("V", [3008, 50257])
def test_duplicate_sequences_in_group(V):
    # identical rows give identical ell when they sit at the same 16-byte alignment (V even
    # here; for odd V the head/vector split differs per row and ell agrees to rounding)
    z, tok, mask, ref, rew = _edge_inputs(4, 3, V, 4)
    z[1], tok[1], ref[1], rew[1] = z[0], tok[0], ref[0], rew[0]
    o, _, _ = _oracle_compare(z, tok, mask, ref, rew, 1.0, 4)
    sl = o.seq_logp.cpu().numpy()
    if V % 8 == 0:
        assert sl[0] == sl[1]
    else:
        assert abs(sl[0] - sl[1]) <= 1e-9 * abs(sl[0])


def test_in_place_dlogits_aliasing():
    w = W("pythia", B=2, K=2, T=3, V=5000)
    inp = H.device_inputs(w, 11)
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, w.N)
    ref = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N)
    lg = inp["logits"].clone()
    out = tba.vargrad_bwd(lg, inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N, dlogits=lg)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def test_token_out_of_range_sets_device_status():
    z, tok, mask, ref, rew = _edge_inputs(2, 2, 100, 2, dtype=torch.float32)
    tok[1, 1] = 100
    with pytest.raises(ValueError, match="device status 1"):
        tba.vargrad_fwd(z.cuda(), tok.cuda(), mask.cuda(), ref.cuda(), rew.cuda(), 1.0, 2, 2, check_status=True)
    tok[1, 1] = -1
    mask[1, 1] = 0  # masked: legal
    tba.vargrad_fwd(z.cuda(), tok.cuda(), mask.cuda(), ref.cuda(), rew.cuda(), 1.0, 2, 2, check_status=True)


def test_all_neg_inf_row_sets_nonfinite_status():
    z, tok, mask, ref, rew = _edge_inputs(2, 2, 64, 2, dtype=torch.float32)
    z[0, 1] = float("-inf")
    with pytest.raises(ValueError, match="device status 2"):
        tba.seq_logprob(z.cuda(), tok.cuda(), mask.cuda(), check_status=True)


def test_zero_groups_rank_gives_zero_partial():
    w = W("toy", B=0)
    inp = H.device_inputs(w, 0)
    o, _ = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], 1.0, 4,
                           8.0)
    assert o.partial.cpu().tolist() == [0.0, 0.0, 0.0]


def test_config_errors_raise():
    z, tok, mask, ref, rew = _edge_inputs(4, 2, 64, 2, dtype=torch.float32)
    args = (z.cuda(), tok.cuda(), mask.cuda(), ref.cuda(), rew.cuda())
    with pytest.raises(tba.TbaError):
        tba.vargrad_fwd(*args, 0.0, 2, 4)
    with pytest.raises(tba.TbaError):
        tba.vargrad_fwd(*args, 1.0, 1, 4)
    with pytest.raises(tba.TbaError):
        tba.vargrad_fwd(*args, 1.0, 3, 4)


# ------------------------------------------------------------------------------- seq_logprob / autograd
def test_seq_logprob_matches_oracle():
    w = W("rhomath", B=2, K=3, T=7, V=32000, len_lo=0, len_hi=7)
    inp = H.device_inputs(w, 3)
    sl, nt = tba.seq_logprob(inp["logits"], inp["tokens"], inp["mask"].bool())
    lg = H.host_logits(w, 3, 0, w.B)
    ell, ntok, _ = O.seq_logprob(lg, inp["host"]["tokens"], inp["host"]["mask"])
    H.assert_seq_close(sl.cpu().numpy(), ell, "seq_logprob")
    np.testing.assert_array_equal(nt.cpu().numpy(), ntok)


def test_autograd_function():
    w = W("pythia", B=2, K=4, T=3, V=2048)
    inp = H.device_inputs(w, 12)
    lg = inp["logits"].clone().requires_grad_(True)
    loss, aux = tba.vargrad_tb_loss(lg, inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                                    return_aux=True)
    (3.0 * loss).backward()
    h = inp["host"]
    ref = O.vargrad_head(H.host_logits(w, 12, 0, w.B), h["tokens"], h["mask"], h["ref_logp"], h["log_reward"],
                         w.beta, w.K, grad_out=3.0)
    H.assert_seq_close([loss.item()], [ref["loss"]], "loss")
    g = lg.grad.double().cpu().numpy()
    for s in range(w.N):
        for t in range(w.T):
            H.assert_dlogits_close(g[s, t], ref["dlogits"][s, t], 6.0 * ref["eps"][s] / w.N, "bf16")


# ------------------------------------------------------------------------------- metamorphic / determinism
def test_determinism_bitwise():
    w = W("pythia", B=2, K=4, T=6)
    inp = H.device_inputs(w, 1)
    a = run_gpu(inp, w)
    b = run_gpu(inp, w)
    assert torch.equal(a[0].seq_logp, b[0].seq_logp) and torch.equal(a[0].partial, b[0].partial)
    assert torch.equal(a[1].view(torch.int16), b[1].view(torch.int16))


def test_group_reward_shift_invariance():
    w = W("redteam", B=3, K=4, T=4)
    inp = H.device_inputs(w, 2)
    a = run_gpu(inp, w)
    inp2 = dict(inp)
    shift = torch.tensor([0.25, -0.5, 1.0], dtype=torch.float64, device="cuda").repeat_interleave(w.K)
    inp2["log_reward"] = inp["log_reward"] + w.beta * shift * 4  # exact binary shifts of r/beta... up to rounding
    b = run_gpu(inp2, w)
    H.assert_seq_close(b[0].resid.cpu().numpy(), a[0].resid.cpu().numpy(), "resid shift", rel=1e-9, abs_=1e-9)
    da, db = a[1].float(), b[1].float()
    assert torch.max(torch.abs(da - db)).item() <= 2 * torch.max(torch.abs(da)).item() * 2 ** -8


def test_vocab_one_and_two():
    for V in (1, 2, 3):
        z, tok, mask, ref, rew = _edge_inputs(4, 3, V, 2, dtype=torch.bfloat16, seed=V)
        _oracle_compare(z, tok, mask, ref, rew, 0.25, 2)


def test_zero_length_responses_shape():
    """seq_len = 0: every response empty; ell = 0, loss from ref/rewards only, no rows."""
    N, K = 4, 2
    z = torch.zeros((N, 0, 7), dtype=torch.bfloat16, device="cuda")
    tok = torch.zeros((N, 0), dtype=torch.int64, device="cuda")
    mask = torch.zeros((N, 0), dtype=torch.uint8, device="cuda")
    ref = torch.tensor([-1.0, -2.0, -3.0, 0.5], dtype=torch.float64, device="cuda")
    rew = torch.tensor([0.0, 1.0, 1.0, 0.0], dtype=torch.float64, device="cuda")
    o, ws = tba.vargrad_fwd(z, tok, mask, ref, rew, 0.5, K, N)
    d = tba.vargrad_bwd(z, tok, mask, ws, o.resid, 2.0 / N)
    torch.cuda.synchronize()
    r = O.vargrad_tb_loss(np.zeros(N), ref.cpu().numpy(), rew.cpu().numpy(), 0.5, K)
    assert o.seq_logp.abs().sum().item() == 0 and o.n_tokens.sum().item() == 0
    H.assert_seq_close([o.partial[0].item()], [r[0]], "loss")
    assert d.shape == (N, 0, 7)


def test_power_of_two_shift_metamorphic():
    """Adding 16 to every logit of a row (exact in bf16 for half-integer logits) leaves the
    log-probs and the gradient unchanged (softmax shift invariance)."""
    g = torch.Generator().manual_seed(3)
    N, T, V, K = 4, 3, 5000, 2
    z = (torch.randint(-16, 17, (N, T, V), generator=g).float() / 2).to(torch.bfloat16)
    zs = (z.float() + 16.0).to(torch.bfloat16)
    assert torch.equal(zs.float() - 16.0, z.float())            # the shift is exact
    tok = torch.randint(0, V, (N, T), generator=g).cuda()
    mask = torch.ones(N, T, dtype=torch.uint8, device="cuda")
    ref = torch.randn(N, generator=g, dtype=torch.float64).cuda() - 30
    rew = torch.rand(N, generator=g, dtype=torch.float64).cuda()
    a, wa = tba.vargrad_fwd(z.cuda(), tok, mask, ref, rew, 0.5, K, N)
    b, wb = tba.vargrad_fwd(zs.cuda(), tok, mask, ref, rew, 0.5, K, N)
    da = tba.vargrad_bwd(z.cuda(), tok, mask, wa, a.resid, 2.0 / N)
    db = tba.vargrad_bwd(zs.cuda(), tok, mask, wb, b.resid, 2.0 / N)
    torch.cuda.synchronize()
    H.assert_seq_close(b.seq_logp.cpu().numpy(), a.seq_logp.cpu().numpy(), "shifted seq_logp", rel=1e-6, abs_=1e-6)
    x, y = da.float(), db.float()
    assert torch.max(torch.abs(x - y)).item() <= 2 * 2 ** -8 * torch.max(torch.abs(x)).item()


def test_sharded_equals_unsharded_on_one_gpu():
    """Whole-group shards run one after another (what ranks do in parallel): per-sequence outputs
    and dlogits are bit-identical to the unsharded run, the partials sum to its loss."""
    w = W("qwen", B=6, K=4, T=3)   # aligned rows: identical per-row arithmetic in every shard
    full = H.device_inputs(w, 4)
    N = w.N
    o, ws = tba.vargrad_fwd(full["logits"], full["tokens"], full["mask"], full["ref_logp"], full["log_reward"], w.beta,
                            w.K, N)
    d = tba.vargrad_bwd(full["logits"], full["tokens"], full["mask"], ws, o.resid, 2.0 / N)
    parts = []
    for g0, g1 in [tba.group_range(w.B, 4, r) for r in range(4)]:
        sl = slice(g0 * w.K, g1 * w.K)
        if g1 == g0:
            continue
        lg = full["logits"][sl].contiguous()
        os_, wss = tba.vargrad_fwd(lg, full["tokens"][sl].contiguous(), full["mask"][sl].contiguous(),
                                   full["ref_logp"][sl].contiguous(), full["log_reward"][sl].contiguous(), w.beta,
                                   w.K, N)
        ds = tba.vargrad_bwd(lg, full["tokens"][sl].contiguous(), full["mask"][sl].contiguous(), wss, os_.resid,
                             2.0 / N)
        torch.cuda.synchronize()
        assert torch.equal(os_.seq_logp, o.seq_logp[sl]) and torch.equal(os_.resid, o.resid[sl])
        assert torch.equal(ds.view(torch.int16), d[sl].view(torch.int16))
        parts.append(os_.partial.cpu().numpy())
    tot = np.sum(parts, axis=0)
    p = o.partial.cpu().numpy()
    assert abs(tot[0] - p[0]) <= 1e-12 * p[0] and tot[1] == p[1] and tot[2] == p[2]


@pytest.mark.parametrize("V,T,dt", [(262144, 2, "bf16"), (131072, 3, "fp32"), (1000, 8192, "bf16")])
def test_extreme_shapes(V, T, dt):
    """Vocabularies past Qwen's (512 KB bf16 / fp32 rows) and very long responses."""
    w = W("qwen", B=1, K=2, T=T, V=V, dtype=dt, len_lo=T // 2, len_hi=T)
    compare_full(w, 3) if V * T <= 2 ** 20 else _compare_sampled(w, 3)


def _compare_sampled(w, seed):
    inp = H.device_inputs(w, seed)
    o, d = run_gpu(inp, w)
    ref = H.oracle_seq_values(w, seed, 0, w.B)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp")
    loss, logz, eps = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, w.K)
    H.assert_seq_close(o.resid.cpu().numpy(), eps, "resid")
    rng = np.random.default_rng(seed)
    mask = ref["mask"]
    for r in rng.choice(np.flatnonzero(mask.reshape(-1)), size=8, replace=False):
        s, t = divmod(int(r), w.T)
        z = syn.logits_rows_f64(seed, w.V, [r], w.dtype)[0]
        want = O.dlogits_row(z, int(ref["tokens"][s, t]), eps[s], w.N)
        got = d[s, t].double().cpu().numpy()
        H.assert_dlogits_close(got, want, 2 * eps[s] / w.N, "bf16" if d.dtype == torch.bfloat16 else "fp32")


@pytest.mark.parametrize("inv_temp", [1.0, 1 / 0.7])
def test_token_logprob_matches_oracle(inv_temp):
    w = W("redteam", B=2, K=3, T=6, len_lo=2, len_hi=6)
    inp = H.device_inputs(w, 9)
    tl = tba.token_logprob(inp["logits"], inp["tokens"], inp["mask"], inv_temp=inv_temp, check_status=True)
    torch.cuda.synchronize()
    lg = H.host_logits(w, 9, 0, w.B) * inv_temp
    h = inp["host"]
    got = tl.cpu().numpy()
    for s in range(w.N):
        for t in range(w.T):
            if h["mask"][s, t]:
                want, _ = O.token_logprob(lg[s, t], int(h["tokens"][s, t]))
                assert abs(got[s, t] - want) <= 1e-5 * max(1.0, abs(want))
            else:
                assert got[s, t] == 0.0
    sl, _ = tba.seq_logprob(inp["logits"], inp["tokens"], inp["mask"])
    if inv_temp == 1.0:
        H.assert_seq_close(tl.sum(1).cpu().numpy(), sl.cpu().numpy(), "sum of token log-probs", rel=1e-9, abs_=1e-9)
