"""Hostile-input parity (GPU vs the fp64 oracle, element by element): rows built to stress the
row kernels' numerics rather than drawn from the workload recipe.

* monotone ramps rising by more than the re-base slack every chunk (a re-base on every chunk,
  the max in the last vector) and falling ramps (the max in the first vector);
* bf16 logits of magnitude 10^2-10^3;
* -inf blocks in middle tiles, rows that are -inf except a few finite entries at the end;
* constant rows (p = 1/V exactly);
* a peak in the last 16-byte vector of a row and at the row's last element;
* fp32 dlogits with |c_seq| ~ 10 (the R9 bar 2e-6*max(1,|c|) at its largest scale).
Every case records max |err| and max err/tol (tests/_harness.RECORD -> $TBA_PARITY_OUT), so the
margin against each bar is on file (profiles/parity_r02.json)."""
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

K = 4
T = 4
N = 2 * K


def _bf16(z):
    return syn.bf16_bits_to_f64(syn.f32_to_bf16_bits(np.asarray(z, np.float32)))


def _row(kind, V, rng):
    v = np.arange(V, dtype=np.float64)
    if kind == "ramp_up":          # +1000 over the row: every chunk's max clears the 6-nat slack
        return -500.0 + 1000.0 * v / (V - 1)
    if kind == "ramp_down":
        return 500.0 - 1000.0 * v / (V - 1)
    if kind == "ramp_up_small":    # a gentle ramp: re-bases far apart, max at the end
        return -8.0 + 16.0 * v / (V - 1)
    if kind == "big300":
        return rng.normal(0.0, 300.0, V)
    if kind == "big1000":
        return np.clip(rng.normal(0.0, 1000.0, V), -3e4, 3e4)
    if kind == "ninf_block":
        z = rng.normal(0.0, 2.0, V)
        a = V // 3
        z[a:a + min(5000, V // 4)] = -np.inf
        return z
    if kind == "ninf_mostly":      # finite only in the last 3 elements and one in the middle
        z = np.full(V, -np.inf)
        z[-3:] = [1.0, -2.0, 0.5]
        z[V // 2] = 3.0
        return z
    if kind == "constant":
        return np.full(V, 3.0)
    if kind == "peak_last_vec":
        z = rng.normal(0.0, 2.0, V)
        z[-5] = 40.0
        return z
    if kind == "peak_last_elem":
        z = rng.normal(0.0, 2.0, V)
        z[-1] = 25.0
        return z
    raise ValueError(kind)


KINDS = ["ramp_up", "ramp_down", "ramp_up_small", "big300", "big1000", "ninf_block", "ninf_mostly", "constant",
         "peak_last_vec", "peak_last_elem"]


def _inputs(V, dtype, seed, kinds, big_c=False):
    rng = np.random.default_rng(seed)
    z = np.empty((N, T, V))
    for s in range(N):
        for t in range(T):
            z[s, t] = _row(kinds[(s * T + t) % len(kinds)], V, rng)
    z = _bf16(z) if dtype == "bf16" else z.astype(np.float32).astype(np.float64)
    tokens = np.empty((N, T), np.int64)
    for s in range(N):
        for t in range(T):
            fin = np.flatnonzero(np.isfinite(z[s, t]))          # a token at a finite logit
            tokens[s, t] = fin[rng.integers(0, len(fin))] if (s + t) % 3 else fin[np.argmax(z[s, t][fin])]
    mask = np.ones((N, T), np.uint8)
    mask[1, 3] = 0
    mask[5, 0] = 0
    ref = rng.normal(-20.0, 5.0, N)
    if big_c:   # residuals of +-40 -> |c| = 2*40/N = 10
        rew = np.tile([40.0, -40.0, 40.0, -40.0], N // 4) + rng.normal(0, 0.1, N)
    else:
        rew = rng.normal(0.0, 1.0, N)
    ref = ref.astype(np.float32).astype(np.float64)
    rew = rew.astype(np.float32).astype(np.float64)
    return z, tokens, mask, ref, rew


def _run(z, tokens, mask, ref, rew, beta, dtype, out_dtype, test, what):
    dev = "cuda"
    lg = torch.from_numpy(z).to(dev, torch.bfloat16 if dtype == "bf16" else torch.float32)
    tk, mk = torch.from_numpy(tokens).to(dev), torch.from_numpy(mask).to(dev)
    rf, rw = torch.from_numpy(ref).to(dev), torch.from_numpy(rew).to(dev)
    o, ws = tba.vargrad_fwd(lg, tk, mk, rf, rw, beta, K, float(N), check_status=True)
    d = tba.vargrad_bwd(lg, tk, mk, ws, o.resid, 2.0 / N, dlogits_dtype=out_dtype)
    torch.cuda.synchronize()
    r = O.vargrad_head(z, tokens, mask, ref, rew, beta, K)
    cfg = f"hostile V={z.shape[-1]} {dtype}->{'bf16' if out_dtype == torch.bfloat16 else 'fp32'}"
    for name, g, want in (("seq_logp", o.seq_logp, r["ell"]), ("log_z", o.log_z, r["log_z"]),
                          ("resid", o.resid, r["eps"])):
        g = g.cpu().numpy()
        rr = H.assert_seq_close(g, want, f"{what} {name}")
        H.record(test, cfg, 0, f"{name} [{what}]", len(g), np.max(np.abs(g - want)), rr)
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), r["n_tok"])
    dd = d.float().cpu().numpy().astype(np.float64)
    od = "bf16" if out_dtype == torch.bfloat16 else "fp32"
    worst_abs, worst_ratio = 0.0, 0.0
    for s in range(N):
        c = 2.0 * r["eps"][s] / N
        for t in range(T):
            H.assert_dlogits_close(dd[s, t], r["dlogits"][s, t], c, od, f"{what} s={s} t={t}")
            if od == "bf16":
                rb = O.round_bf16(r["dlogits"][s, t])
                ratio = np.abs(dd[s, t] - rb) / O.bf16_ulp(rb)
                ftz = 2.0 ** -126 * max(1.0, abs(c))
                ratio[(np.abs(dd[s, t]) < ftz) & (np.abs(rb) < ftz)] = 0.0
            else:
                ratio = np.abs(dd[s, t] - r["dlogits"][s, t]) / (2e-6 * max(1.0, abs(c)))
            worst_ratio = max(worst_ratio, float(ratio.max()))
            worst_abs = max(worst_abs, float(np.abs(dd[s, t] - r["dlogits"][s, t]).max()))
    H.record(test, cfg, 0, f"dlogits [{what}]", N * T, worst_abs, worst_ratio,
             tol="1 bf16 ulp" if od == "bf16" else "2e-6*max(1,|c|)", max_abs_c=float(np.max(np.abs(2 * r["eps"] / N))))
    return worst_ratio


@pytest.mark.parametrize("V", [32000, 50257, 152064])
def test_hostile_rows_bf16(V):
    z, tokens, mask, ref, rew = _inputs(V, "bf16", V, KINDS)
    _run(z, tokens, mask, ref, rew, 1.0, "bf16", torch.bfloat16, "hostile_bf16", "mixed hostile rows")


@pytest.mark.parametrize("V", [1000, 32000, 152064])
def test_hostile_rows_fp32_out_moderate(V):
    """fp32 dlogits on the rows whose logits stay in a realistic range (|z - max| <~ 64 on the
    mass of the softmax): the R9 bar must hold as written."""
    kinds = ["ramp_up_small", "ninf_block", "ninf_mostly", "constant", "peak_last_vec", "peak_last_elem"]
    z, tokens, mask, ref, rew = _inputs(V, "fp32", V + 1, kinds)
    _run(z, tokens, mask, ref, rew, 1.0, "fp32", torch.float32, "hostile_fp32", "moderate rows")


@pytest.mark.parametrize("V", [1000, 50257])
def test_fp32_dlogits_large_c(V):
    """|c_seq| ~ 10 with fp32 logits and dlogits, peaked rows (p ~ 1 at the max): the
    2e-6*max(1,|c|) bar at its largest absolute scale; the margin is recorded."""
    kinds = ["peak_last_vec", "peak_last_elem", "constant", "ramp_up_small"]
    z, tokens, mask, ref, rew = _inputs(V, "fp32", 7 * V, kinds, big_c=True)
    _run(z, tokens, mask, ref, rew, 1.0, "fp32", torch.float32, "hostile_large_c", "|c|~10 fp32")


def test_hostile_bf16_in_fp32_out_large_c():
    z, tokens, mask, ref, rew = _inputs(152064, "bf16", 3, ["peak_last_vec", "ramp_up_small", "ninf_block",
                                                              "peak_last_elem"], big_c=True)
    _run(z, tokens, mask, ref, rew, 1.0, "bf16", torch.float32, "hostile_large_c", "bf16 in, fp32 out, |c|~10")


@pytest.mark.parametrize("peak", [16.0, 24.0])
def test_confident_sequences(peak):
    """Confident sequences, the common case of a trained policy: every token's logit stands `peak`
    above N(0, 1) noise at V = 32000, so 1 - p_y ~ V e^(0.5 - peak) (5e-3 and 2e-6) and a 256-token
    response has |ell| of 1e-3 .. 1: log p_y and 1 - p_y must keep their RELATIVE accuracy (R24;
    summing the token's term with the others in fp32 would lose ~2e-7 of p_y per token, 1e-4 of ell
    here). Every per-sequence value, and dlogits including each row's token entry, against the oracle."""
    V, Tc, Kc = 32000, 256, 4
    Nc = 2 * Kc
    rng = np.random.default_rng(int(peak))
    z = rng.normal(0.0, 1.0, (Nc, Tc, V))
    tokens = rng.integers(0, V, (Nc, Tc))
    z[np.arange(Nc)[:, None], np.arange(Tc)[None, :], tokens] += peak
    z = _bf16(z)
    mask = np.ones((Nc, Tc), np.uint8)
    mask[3, 200:] = 0
    ref = (rng.normal(0.0, 1e-3, Nc)).astype(np.float32).astype(np.float64)
    rew = (rng.normal(0.0, 1.0, Nc)).astype(np.float32).astype(np.float64)
    dev = "cuda"
    lg = torch.from_numpy(z).to(dev, torch.bfloat16)
    tk, mk = torch.from_numpy(tokens).to(dev), torch.from_numpy(mask).to(dev)
    o, ws = tba.vargrad_fwd(lg, tk, mk, torch.from_numpy(ref).to(dev), torch.from_numpy(rew).to(dev), 1.0, Kc,
                            float(Nc), check_status=True)
    d = tba.vargrad_bwd(lg, tk, mk, ws, o.resid, 2.0 / Nc)
    torch.cuda.synchronize()
    r = O.vargrad_head(z, tokens, mask, ref, rew, 1.0, Kc)
    sl = o.seq_logp.cpu().numpy()
    # the literal bar (rel 1e-4, abs 1e-5) is loose at |ell| ~ 1e-3: hold the sequence log-probs to
    # 1e-5 RELATIVE as well, which summing through fp32 with the token's term included would miss
    rr = H.assert_close_tol(sl, r["ell"], 1e-5 * np.abs(r["ell"]) + 1e-12, f"confident peak {peak} seq_logp")
    H.record("hostile_confident", f"V=32000 peak={peak}", 0, "seq_logp (rel 1e-5)", Nc, np.max(np.abs(sl - r["ell"])),
             rr, ell_range=[float(np.min(r["ell"])), float(np.max(r["ell"]))])
    dd = d.float().cpu().numpy().astype(np.float64)
    worst = 0.0
    for s in range(Nc):
        c = 2.0 * r["eps"][s] / Nc
        for t in range(Tc):
            H.assert_dlogits_close(dd[s, t], r["dlogits"][s, t], c, "bf16", f"confident s={s} t={t}")
            if mask[s, t]:
                y = int(tokens[s, t])
                rb = O.round_bf16(np.array([r["dlogits"][s, t, y]]))[0]
                worst = max(worst, abs(dd[s, t, y] - rb) / O.bf16_ulp(np.array([rb]))[0])
    H.record("hostile_confident", f"V=32000 peak={peak}", 0, "dlogits token entries (ulp)", Nc * Tc, 0.0, worst)
