"""The one-launch fused schedule (tba_tb_loss_fused) reproduces the
two-call path bit for bit, for every shape class, lookahead and variant."""
import dataclasses
import os

import numpy as np
import pytest

import tba_synth as syn

from . import _harness as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2503_18929_b200 as tba  # noqa: E402


def W(name, **kw):
    return dataclasses.replace(syn.WORKLOADS[name], **kw)


CASES = [
    ("toy", W("toy")),
    ("rt_ragged_unaligned", W("redteam", B=6, K=4, T=9, len_lo=0, len_hi=9)),
    ("pythia_full", syn.WORKLOADS["pythia"]),
    ("rhomath_small_ragged", W("rhomath", B=5, K=4, T=40, len_lo=3, len_hi=40)),
    ("qwen_small", W("qwen", B=3, K=4, T=8)),
]


def _two_call(inp, w, inv_temp=1.0, lz=None, dl_dtype=None):
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, w.N, inv_temp=inv_temp, log_z_param=lz)
    r = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N, inv_temp=inv_temp,
                        log_z_param=lz, K=w.K, dlogits_dtype=dl_dtype)
    d, dz = (r, None) if lz is None else r
    return o, d, dz


@pytest.mark.parametrize("name,w", CASES, ids=[c[0] for c in CASES])
def test_fused_equals_two_call(name, w):
    inp = H.device_inputs(w, 7)
    a, da, _ = _two_call(inp, w)
    b, ws, db, _ = tba.vargrad_fused(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"],
                                     w.beta, w.K, float(w.N), check_status=True)
    torch.cuda.synchronize()
    for f in ("seq_logp", "n_tokens", "log_z", "resid", "partial"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    assert torch.equal(da.view(torch.int16) if da.dtype == torch.bfloat16 else da,
                       db.view(torch.int16) if db.dtype == torch.bfloat16 else db)


@pytest.mark.parametrize("D", ["1", "2", "64"])
def test_fused_lookahead_values(D, monkeypatch):
    # the lookahead only changes the schedule; D is read once per process, so run a subprocess
    import subprocess
    import sys
    code = (
        "import dataclasses, torch, tba_synth as syn, paper_2503_18929_b200 as tba\n"
        "from tests import _harness as H\n"
        "w = dataclasses.replace(syn.WORKLOADS['pythia'], B=12)\n"
        "inp = H.device_inputs(w, 3)\n"
        "o, ws = tba.vargrad_fwd(inp['logits'], inp['tokens'], inp['mask'], inp['ref_logp'], inp['log_reward'], w.beta, w.K, w.N)\n"
        "d = tba.vargrad_bwd(inp['logits'], inp['tokens'], inp['mask'], ws, o.resid, 2.0 / w.N)\n"
        "b, _, db, _ = tba.vargrad_fused(inp['logits'], inp['tokens'], inp['mask'], inp['ref_logp'], inp['log_reward'], w.beta, w.K, float(w.N))\n"
        "torch.cuda.synchronize()\n"
        "assert torch.equal(o.partial, b.partial) and torch.equal(d.view(torch.int16), db.view(torch.int16))\n"
        "print('ok')\n")
    env = dict(os.environ, TBA_FUSED_D=D)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_fused_variants_and_fp32_out_and_alias():
    w = W("pythia", B=3, K=4, T=6, V=5003)
    inp = H.device_inputs(w, 9)
    lz = torch.tensor([-20.0, 3.0, 40.0], dtype=torch.float64, device="cuda")
    a, da, dza = _two_call(inp, w, inv_temp=1 / 0.7, lz=lz, dl_dtype=torch.float32)
    b, _, db, dzb = tba.vargrad_fused(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"],
                                      w.beta, w.K, float(w.N), dlogits_dtype=torch.float32, inv_temp=1 / 0.7,
                                      log_z_param=lz)
    torch.cuda.synchronize()
    assert torch.equal(a.resid, b.resid) and torch.equal(da, db) and torch.equal(dza, dzb)
    # in place: dlogits overwrite the logits they are computed from
    a2, da2, _ = _two_call(inp, w)
    lg = inp["logits"].clone()
    b2, _, db2, _ = tba.vargrad_fused(lg, inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                                      float(w.N), dlogits=lg)
    torch.cuda.synchronize()
    assert torch.equal(a2.partial, b2.partial) and torch.equal(da2.view(torch.int16), lg.view(torch.int16))


def test_loss_and_grad_api():
    w = W("redteam", B=4, K=8, T=5)
    inp = H.device_inputs(w, 1)
    loss, d = tba.vargrad_tb_loss_and_grad(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                           inp["log_reward"], w.beta, w.K)
    lg = inp["logits"].clone().requires_grad_(True)
    l2 = tba.vargrad_tb_loss(lg, inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K)
    l2.backward()
    assert loss.item() == l2.item()
    assert torch.equal(d.view(torch.int16), lg.grad.view(torch.int16))


@pytest.mark.parametrize("name,w", CASES, ids=[c[0] for c in CASES])
def test_deferred_scale_matches_oracle(name, w):
    """G from the single-pass deferred kernel, scaled by (2/N) eps_s, is the oracle's dlogits
    (fp32 G: 2e-6 max(1,|c|); bf16 G: within 2 bf16 ulps of the oracle — G and c.G each round once)."""
    from oracle import tba_oracle as O
    inp = H.device_inputs(w, 5)
    h = inp["host"]
    dt = torch.float32 if w.dtype == "fp32" else torch.bfloat16
    o, ws, G = tba.vargrad_fwd_deferred(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                        inp["log_reward"], w.beta, w.K, float(w.N), g_dtype=torch.float32,
                                        check_status=True)
    a, _ = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                           w.K, w.N)
    torch.cuda.synchronize()
    # different threads-per-row => different fp32 summation order: agree to rounding, both match the oracle
    H.assert_seq_close(o.resid.cpu().numpy(), a.resid.cpu().numpy(), "deferred resid vs two-call", rel=1e-5,
                       abs_=1e-6)
    eps = o.resid.cpu().numpy()
    rng = np.random.default_rng(0)
    rows = rng.choice(w.N * w.T, size=min(24, w.N * w.T), replace=False)
    Gh = G.view(-1, w.V)
    for r in rows:
        s_, t = divmod(int(r), w.T)
        got = Gh[r].double().cpu().numpy() * (2 * eps[s_] / w.N)
        if h["mask"][s_, t]:
            z = syn.logits_rows_f64(5, w.V, [r], w.dtype)[0]
            want = O.dlogits_row(z, int(h["tokens"][s_, t]), eps[s_], w.N)
            H.assert_dlogits_close(got, want, 2 * eps[s_] / w.N, "fp32", f"row {r}")
        else:
            assert np.all(got == 0)
    # bf16 G: also valid
    o2, _, G2 = tba.vargrad_fwd_deferred(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                         inp["log_reward"], w.beta, w.K, float(w.N))
    torch.cuda.synchronize()
    assert torch.allclose(G2.double(), G.double(), rtol=2 ** -8, atol=1e-30)


@pytest.mark.parametrize("V", [5003, 50257, 80000])
def test_deferred_both_row_classes(V):
    """The deferred kernel's two row classes (<= 128 KB rows: 256 threads; longer: 512 threads with 8
    vectors in flight) give the oracle's dlogits once the row scale is applied."""
    w = W("redteam", B=2, K=4, T=5, V=V, len_lo=1, len_hi=5)   # ragged; odd row length at 50257
    inp = H.device_inputs(w, 2)
    o, _, G = tba.vargrad_fwd_deferred(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                       inp["log_reward"], w.beta, w.K, float(w.N), g_dtype=torch.float32,
                                       check_status=True)
    torch.cuda.synchronize()
    from oracle import tba_oracle as O
    h = inp["host"]
    ref = O.vargrad_head(H.host_logits(w, 2, 0, w.B), h["tokens"], h["mask"], h["ref_logp"], h["log_reward"], w.beta,
                         w.K)
    eps = o.resid.cpu().numpy()
    H.assert_seq_close(eps, ref["eps"], "resid")
    g = G.double().cpu().numpy()
    for s_ in range(w.N):
        for t in range(w.T):
            H.assert_dlogits_close(g[s_, t] * 2 * eps[s_] / w.N, ref["dlogits"][s_, t], 2 * eps[s_] / w.N, "fp32")


def test_cuda_graph_capture_replays_bitwise():
    w = W("redteam", B=4, K=8, T=5)
    inp = H.device_inputs(w, 6)
    ws = torch.empty(tba.workspace_bytes(w.N, w.T), dtype=torch.uint8, device="cuda")
    out = tba.ops._Fwd(w.N, w.K, torch.device("cuda"))
    d = torch.empty_like(inp["logits"])

    def step():
        tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                        float(w.N), workspace=ws, out=out, check_status=False)
        tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, out.resid, 2.0 / w.N, dlogits=d)

    step()
    torch.cuda.synchronize()
    ref_d, ref_p = d.clone(), out.partial.clone()
    d.zero_()
    out.partial.zero_()
    g = tba.CapturedStep(step)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.partial, ref_p) and torch.equal(d.view(torch.int16), ref_d.view(torch.int16))


@pytest.mark.parametrize("name,seed,sched", [("pythia", 5, "fused"), ("redteam", 6, "fused"),
                                             ("pythia", 8, "pipelined")])
def test_one_call_schedules_against_oracle(name, seed, sched):
    """The one-launch / pipelined schedules compared with the fp64 ORACLE directly (not only with
    the two-call CUDA path): every per-sequence value, the loss and every dlogits row."""
    import numpy as np

    from oracle import tba_oracle as O
    w = syn.WORKLOADS[name]
    inp = H.device_inputs(w, seed)
    call = tba.vargrad_fused if sched == "fused" else tba.vargrad_pipelined
    o, _, d, _ = call(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta, w.K,
                      float(w.N), check_status=True)
    torch.cuda.synchronize()
    ref = H.oracle_seq_values(w, seed, 0, w.B)
    test = f"{sched}_vs_oracle"
    sl = o.seq_logp.cpu().numpy()
    H.record(test, name, seed, "seq_logp", w.N, np.max(np.abs(sl - ref["ell"])),
             H.assert_seq_close(sl, ref["ell"], "seq_logp"))
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), ref["n_tok"])
    loss, logz, eps = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, w.K)
    for q, g, want in (("log_z", o.log_z, logz), ("resid", o.resid, eps), ("loss", o.partial[:1], [loss])):
        g = g.cpu().numpy()
        H.record(test, name, seed, q, len(g), np.max(np.abs(g - want)), H.assert_seq_close(g, want, q))
    rows = np.flatnonzero(ref["mask"].reshape(-1))
    n, ma, mr = H.compare_dlogits_rows(d, w, seed, rows, 0, ref["tokens"].reshape(-1), np.repeat(eps, w.T), w.N,
                                       what=test)
    H.record(test, name, seed, "dlogits (every valid row)", n, ma, mr, tol="1 bf16 ulp")


@pytest.mark.parametrize("V,dtype,g_dtype", [(80001, "bf16", "fp32"), (80001, "bf16", "bf16"), (76000, "bf16", "fp32"),
                                             (50304, "fp32", "fp32"), (33001, "bf16", "fp32")])
def test_deferred_token_regions_and_alignment(V, dtype, g_dtype):
    """Every region of the deferred kernel's row split holds the sampled token somewhere in the batch:
    the scalar head and tail (odd V: rows start at every 2-byte offset), the shared-memory stash part
    (the row's first 96 KB), the L2 part, the last element; G rows whose 16-byte alignment differs from
    the logits row (fp32 G of odd-V bf16 rows) take the scalar fallback. Each G row times (2/N) eps_s
    is the oracle's dlogits row (App. A)."""
    from oracle import tba_oracle as O
    w = W("redteam", B=2, K=4, T=6, V=V, dtype=dtype, len_lo=1, len_hi=6)
    inp = H.device_inputs(w, 9)
    h = inp["host"]
    esz = 2 if dtype == "bf16" else 4
    stash_elems = 96 * 1024 // esz
    picks = [p for p in [0, 1, 3, 7, 8, stash_elems - 1, stash_elems, stash_elems + 5, V // 2, V - 9, V - 2, V - 1]
             if p < V]
    tok = h["tokens"].copy()
    for i in range(tok.size):
        tok.flat[i] = picks[i % len(picks)] if i % 5 else tok.flat[i]
    h["tokens"] = tok
    inp["tokens"] = torch.from_numpy(tok).cuda()
    gdt = torch.float32 if g_dtype == "fp32" else torch.bfloat16
    o, _, G = tba.vargrad_fwd_deferred(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                       inp["log_reward"], w.beta, w.K, float(w.N), g_dtype=gdt, check_status=True)
    torch.cuda.synchronize()
    ref = O.vargrad_head(H.host_logits(w, 9, 0, w.B), h["tokens"], h["mask"], h["ref_logp"], h["log_reward"], w.beta,
                         w.K)
    eps = o.resid.cpu().numpy()
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp")
    H.assert_seq_close(eps, ref["eps"], "resid")
    g = G.double().cpu().numpy()
    for s_ in range(w.N):
        c = 2 * eps[s_] / w.N
        for t in range(w.T):
            if not h["mask"][s_, t]:
                assert np.all(g[s_, t] == 0)
            elif g_dtype == "fp32":
                H.assert_dlogits_close(g[s_, t] * c, ref["dlogits"][s_, t], c, "fp32", f"row {s_},{t}")
            else:  # bf16 G = bf16(G_exact): within one bf16 ulp of the oracle's dlogits / c
                want = ref["dlogits"][s_, t] / c
                ok = np.abs(g[s_, t] - want) <= O.bf16_ulp(O.round_bf16(want)) + 2.0 ** -126
                assert ok.all(), (s_, t, np.flatnonzero(~ok)[:5])
