"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(SURVEY §8(d) oracle-coverage plan).

* toy, Pythia and red-teaming: every per-sequence value and EVERY dlogits row against the
  fp64 oracle;
* RhoMath and the Qwen per-GPU shard: every per-sequence value (all groups), dlogits on 4096
  seeded random valid rows plus every row of two whole groups;
* the paper's own table shapes and Table 5's MATH shard: every per-sequence value of the
  groups they hold, sampled dlogits rows.
Properties that hold at any size (loss = sum eps^2 / N, sum_v dlogits = 0, masked rows zero,
group permutation / reward-shift metamorphics, bitwise determinism) are checked on the full
outputs. Every comparison's maxima go to tests/_harness.RECORD (-> $TBA_PARITY_OUT)."""
import numpy as np
import pytest

import tba_synth as syn
from oracle import tba_oracle as O

from . import _harness as H

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2503_18929_b200 as tba  # noqa: E402


def run_full(w, seed, g0=0, ng=None):
    ng = w.B if ng is None else ng
    inp = H.device_inputs(w, seed, g0, ng)
    N = ng * w.K
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, float(N), check_status=True)
    d = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / N)
    torch.cuda.synchronize()
    return inp, o, d


def check_seq_values(test, w, seed, o, g0, ng, N):
    """Every per-sequence value of groups g0..g0+ng-1 (ell, n_tok, log Z, eps) and the loss of
    those groups against the oracle. Returns the oracle dict (eps_global, tokens, mask...)."""
    K = w.K
    ref = H.oracle_seq_values(w, seed, g0, ng)
    s = slice(g0 * K, (g0 + ng) * K)
    sl, nt = o.seq_logp.cpu().numpy()[s], o.n_tokens.cpu().numpy()[s]
    lz, eps = o.log_z.cpu().numpy()[g0:g0 + ng], o.resid.cpu().numpy()[s]
    r = H.assert_seq_close(sl, ref["ell"], f"{test} seq_logp")
    H.record(test, w.name, seed, "seq_logp", len(sl), np.max(np.abs(sl - ref["ell"])), r)
    np.testing.assert_array_equal(nt, ref["n_tok"])                       # token counts: bit-exact
    H.record(test, w.name, seed, "n_tokens (bit-exact)", len(nt), 0.0, 0.0)
    loss_g, logz_g, eps_g = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, K, n_global=N)
    tz, te = H.seq_tols(ref["ell"], K)              # propagated from the ell bar (reading R23)
    r = H.assert_close_tol(lz, logz_g, tz, f"{test} log_z")
    H.record(test, w.name, seed, "log_z", len(lz), np.max(np.abs(lz - logz_g)), r, tol="propagated from ell (R23)")
    r = H.assert_close_tol(eps, eps_g, te, f"{test} resid")
    H.record(test, w.name, seed, "resid", len(eps), np.max(np.abs(eps - eps_g)), r, tol="propagated from ell (R23)")
    if ng * K == o.resid.shape[0]:                                        # the whole call: the loss too
        p0 = o.partial[0].item()
        r = H.assert_seq_close([p0], [loss_g], f"{test} loss")
        H.record(test, w.name, seed, "loss", 1, abs(p0 - loss_g), r)
    ref["eps_g"] = eps_g
    return ref


def check_dlogits(test, w, seed, d, rows_local, tokens_flat, eps_of_row, N, what):
    n, ma, mr = H.compare_dlogits_rows(d, w, seed, rows_local, 0, tokens_flat, eps_of_row, N, what=f"{test} {what}")
    H.record(test, w.name, seed, f"dlogits ({what})", n, ma, mr,
             tol="1 bf16 ulp" if d.dtype == torch.bfloat16 else "2e-6*max(1,|c|)")


def check_properties(w, inp, o, d, n_rows=64, seed=0):
    eps = o.resid.cpu().numpy()
    N = len(eps)
    p = o.partial.cpu().numpy()
    assert abs(p[0] - np.sum(eps * eps) / N) <= 1e-12 * max(1.0, p[0])       # Eq. 5 over the whole shard
    assert p[1] == N and p[2] == N // w.K
    K = w.K
    for i in range(N // K):                                                   # sum_j eps = 0
        assert abs(eps[i * K:(i + 1) * K].sum()) <= 1e-9 * max(1.0, np.abs(eps[i * K:(i + 1) * K]).max())
    mask = inp["mask"].cpu().numpy()
    rng = np.random.default_rng(seed)
    flat = d.view(-1, w.V)
    rows = rng.choice(N * w.T, size=min(n_rows, N * w.T), replace=False)
    for r in rows:
        row = flat[r].float()
        if mask.reshape(-1)[r]:
            c = abs(2 * eps[r // w.T] / N)
            assert abs(row.double().sum().item()) <= 4e-3 * c + 1e-6             # sum_v (onehot - p) = 0
        else:
            assert torch.count_nonzero(row).item() == 0                         # masked rows are zero
    masked = np.flatnonzero(mask.reshape(-1) == 0)
    for i in range(0, len(masked), 4096):                                     # every masked row is +0
        idx = torch.from_numpy(masked[i:i + 4096]).to(d.device)
        assert torch.count_nonzero(flat.index_select(0, idx).view(torch.int16)).item() == 0


def _row_plan(w, seed, mask_flat, whole_groups, n_random):
    """Local valid rows: every row of `whole_groups` plus n_random seeded random valid rows."""
    valid = np.flatnonzero(mask_flat)
    gr = w.K * w.T
    rows = [valid[(valid >= g * gr) & (valid < (g + 1) * gr)] for g in whole_groups]
    rng = np.random.default_rng(1000 + seed)
    rows.append(rng.choice(valid, size=min(n_random, len(valid)), replace=False))
    return np.unique(np.concatenate(rows))


@pytest.mark.parametrize("name,seed", [("toy", 0), ("pythia", 0), ("redteam", 1)])
def test_full_compare_every_value_and_row(name, seed):
    """Toy, Pythia and red-teaming compared in full: all sequences, every dlogits row."""
    w = syn.WORKLOADS[name]
    test = f"full_{name}"
    inp, o, d = run_full(w, seed)
    ref = check_seq_values(test, w, seed, o, 0, w.B, w.N)
    mask_flat = ref["mask"].reshape(-1)
    eps_row = np.repeat(ref["eps_g"], w.T)
    check_dlogits(test, w, seed, d, np.flatnonzero(mask_flat), ref["tokens"].reshape(-1), eps_row, w.N,
                  "every valid row")
    check_properties(w, inp, o, d)


@pytest.mark.parametrize("name,seed,groups", [("rhomath", 2, [0, 31]), ("qwen_shard", 0, [2, 7])])
def test_large_all_sequences_plus_rows(name, seed, groups):
    """RhoMath and the Qwen shard: every per-sequence value; dlogits on 4096 seeded random
    valid rows plus every row of two whole groups."""
    w = syn.WORKLOADS[name]
    test = f"large_{name}"
    inp, o, d = run_full(w, seed)
    ref = check_seq_values(test, w, seed, o, 0, w.B, w.N)
    mask_flat = ref["mask"].reshape(-1)
    rows = _row_plan(w, seed, mask_flat, groups, 4096)
    eps_row = np.repeat(ref["eps_g"], w.T)
    check_dlogits(test, w, seed, d, rows, ref["tokens"].reshape(-1), eps_row, w.N,
                  f"groups {groups} whole + 4096 random rows")
    check_properties(w, inp, o, d, n_rows=32)
    if name == "qwen_shard":  # bitwise determinism of a second run over the same buffers
        o2, ws2 = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"],
                                  w.beta, w.K, float(w.N))
        assert torch.equal(o2.seq_logp, o.seq_logp) and torch.equal(o2.partial, o.partial)
        d2 = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws2, o2.resid, 2.0 / w.N)
        assert torch.equal(d2.view(torch.int16), d.view(torch.int16))


@pytest.mark.parametrize("name,seed", [("pythia", 1), ("pythia", 2), ("redteam", 0), ("redteam", 2),
                                       ("rhomath", 0), ("rhomath", 1), ("qwen_shard", 1), ("qwen_shard", 2)])
def test_parity_seeds_sequence_values(name, seed):
    """Parity seeds {0, 1, 2}: every per-sequence value and the loss, plus 512
    random dlogits rows, on the other seeds (the Qwen shard's seed 0 is test_large_all_sequences_plus_rows)."""
    w = syn.WORKLOADS[name]
    test = f"seeds_{name}"
    inp, o, d = run_full(w, seed)
    ref = check_seq_values(test, w, seed, o, 0, w.B, w.N)
    rows = _row_plan(w, seed, ref["mask"].reshape(-1), [], 512)
    check_dlogits(test, w, seed, d, rows, ref["tokens"].reshape(-1), np.repeat(ref["eps_g"], w.T), w.N,
                  "512 random rows")


def test_qwen_group_metamorphic_permutation_and_shift():
    """Permuting the K samples of a group permutes every output; adding beta*c to one
    group's log-rewards leaves residuals and dlogits unchanged (no oracle needed)."""
    w = syn.WORKLOADS["qwen_group"]
    inp, o, d = run_full(w, 4)
    K, N = w.K, w.N
    perm = torch.tensor([3, 0, 7, 1, 6, 2, 5, 4], device="cuda")
    pin = {k: v[perm] for k, v in inp.items() if k != "host"}
    pin["logits"] = pin["logits"].contiguous()
    o2, ws2 = tba.vargrad_fwd(pin["logits"], pin["tokens"], pin["mask"], pin["ref_logp"], pin["log_reward"], w.beta,
                              K, float(N))
    assert torch.equal(o2.seq_logp, o.seq_logp[perm]) and torch.equal(o2.n_tokens, o.n_tokens[perm])
    H.assert_seq_close(o2.resid.cpu().numpy(), o.resid[perm].cpu().numpy(), "permuted resid", rel=1e-12, abs_=1e-12)
    del pin, ws2
    torch.cuda.empty_cache()
    rew2 = inp["log_reward"] + w.beta * 0.75
    o3, ws3 = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], rew2, w.beta, K, float(N))
    H.assert_seq_close(o3.resid.cpu().numpy(), o.resid.cpu().numpy(), "shifted resid", rel=1e-9, abs_=1e-9)


@pytest.mark.parametrize("name,seed", [("gsm8k_t3", 0), ("gsm8k_k40", 1), ("tldr_t4", 2)])
def test_paper_table_batch_shapes_full(name, seed):
    """The paper's own batch shapes (Tables 3 and 4, the K = 40 ablation) at full size: every
    per-sequence value, 1024 random dlogits rows plus every row of group 0."""
    w = syn.WORKLOADS[name]
    test = f"paper_{name}"
    inp, o, d = run_full(w, seed)
    ref = check_seq_values(test, w, seed, o, 0, w.B, w.N)
    rows = _row_plan(w, seed, ref["mask"].reshape(-1), [0], 1024)
    check_dlogits(test, w, seed, d, rows, ref["tokens"].reshape(-1), np.repeat(ref["eps_g"], w.T), w.N,
                  "group 0 whole + 1024 random rows")
    check_properties(w, inp, o, d)


def test_math_t5_two_groups_ragged_2048():
    """Table 5's MATH shape (K = 16, responses up to 2048 tokens, V = 152064): two whole groups
    (20 GB of logits), every per-sequence value, 1024 random dlogits rows."""
    w = syn.WORKLOADS["math_t5_shard"]
    test = "paper_math_t5"
    inp, o, d = run_full(w, 3, 0, 2)
    ref = check_seq_values(test, w, 3, o, 0, 2, 2 * w.K)
    rows = _row_plan(w, 3, ref["mask"].reshape(-1), [], 1024)
    check_dlogits(test, w, 3, d, rows, ref["tokens"].reshape(-1), np.repeat(ref["eps_g"], w.T), 2 * w.K,
                  "1024 random rows")
    check_properties(w, inp, o, d, n_rows=32)


@pytest.mark.parametrize("name,seed,mode", [("qwen_shard", 0, "clip"), ("rhomath", 1, "icepop")])
def test_tbap_full_size(name, seed, mode):
    """TBA' (Eq. 16) at full size in bench.py's configuration: every
    per-sequence value (ell, A), every per-token coefficient w(lambda_t) A_j, the surrogate loss,
    and dlogits on 4096 seeded random valid rows plus every row of one whole group."""
    w = syn.WORKLOADS[name]
    test = f"tbap_{name}"
    lo, hi = (0.0, 8.0) if mode == "clip" else (0.5, 2.0)
    inp = H.device_inputs(w, seed)
    gen = torch.from_numpy(syn.gen_logp(w, seed, 0, w.N)).cuda()
    n_tok = float(int(inp["host"]["mask"].sum()))
    o, ws = tba.tbap_fwd(inp["logits"], inp["tokens"], inp["mask"], gen, inp["ref_logp"], inp["log_reward"], w.beta,
                         w.K, mode, lo, hi, n_tok, check_status=True)
    d = tba.tbap_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.coef, n_tok)
    torch.cuda.synchronize()
    lp, gi = H.oracle_token_lp(w, seed, 0, w.B)
    ref = O.tbap_coefficients(lp, gi["mask"], gen.cpu().numpy(), gi["ref_logp"], gi["log_reward"], w.beta, w.K, mode,
                              lo, hi, int(n_tok))
    sl = o.seq_logp.cpu().numpy()
    H.record(test, name, seed, "seq_logp", w.N, np.max(np.abs(sl - ref["ell"])), H.assert_seq_close(sl, ref["ell"], "ell"))
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), ref["n_tok"])
    adv = o.adv.cpu().numpy()
    # A_j inherits ell's bar through beta (log Lambda_j - mean log Lambda): R23 with the factor beta
    tz, te = H.seq_tols(ref["ell"], w.K)
    H.record(test, name, seed, "adv", w.N, np.max(np.abs(adv - ref["adv"])),
             H.assert_close_tol(adv, ref["adv"], w.beta * te, "adv"), tol="beta x propagated (R23)")
    coef = o.coef.cpu().numpy().astype(np.float64)
    m = gi["mask"] == 1
    # coef is stored in fp32: one fp32 rounding of w(lambda) A plus lambda's sensitivity to lp's error
    ctol = np.abs(ref["coef"]) * (2.0 ** -23) + w.beta * np.repeat(te, w.T).reshape(w.N, w.T) * np.maximum(
        1.0, np.abs(np.where(m, ref["coef"], 0.0)))
    r = H.assert_close_tol(coef[m], ref["coef"][m], ctol[m], "coef")
    H.record(test, name, seed, "coef (every valid token)", int(m.sum()), np.max(np.abs(coef[m] - ref["coef"][m])), r)
    p0 = o.partial[0].item()
    H.record(test, name, seed, "loss", 1, abs(p0 - ref["loss"]), H.assert_seq_close([p0], [ref["loss"]], "loss"))
    rows = _row_plan(w, seed, gi["mask"].reshape(-1), [1], 4096)
    # the oracle's own coefficients (fp64) scale the oracle rows; the GPU's fp32 coef differs by ~2^-24
    n, ma, mr = H.compare_dlogits_rows(d, w, seed, rows, 0, gi["tokens"].reshape(-1), ref["coef"].reshape(-1),
                                       int(n_tok), what=f"{test} dlogits", kind="tbap")
    H.record(test, name, seed, "dlogits (group 1 whole + 4096 random rows)", n, ma, mr, tol="1 bf16 ulp")


def test_variants_full_size_temperature_and_learned_log_z():
    """NEXT 4 at the Qwen shard in bench.py's configuration: log pi = log softmax(z / 0.7) and a
    learned log Z(x_i) (Eq. 3): every per-sequence value, the residuals, dL/dlog Z, the loss and
    dlogits on 4096 seeded random valid rows plus every row of one whole group."""
    w = syn.WORKLOADS["qwen_shard"]
    seed, a = 5, 1.0 / 0.7
    test = "variants_qwen_shard"
    inp = H.device_inputs(w, seed)
    lz = np.random.default_rng(77).normal(-40.0, 5.0, w.B)          # the learned per-prompt log Z (an input)
    lz_t = torch.from_numpy(lz).cuda()
    o, ws = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                            w.K, float(w.N), check_status=True, inv_temp=a, log_z_param=lz_t)
    d, dlz = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws, o.resid, 2.0 / w.N, inv_temp=a,
                             log_z_param=lz_t, K=w.K)
    torch.cuda.synchronize()
    ref = H.oracle_seq_values(w, seed, 0, w.B, inv_temp=a)
    sl = o.seq_logp.cpu().numpy()
    H.record(test, w.name, seed, "seq_logp (inv_temp 1/0.7)", w.N, np.max(np.abs(sl - ref["ell"])),
             H.assert_seq_close(sl, ref["ell"], "seq_logp"))
    loss, _, eps = O.tb_learned_z_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, w.K, lz, w.N)
    _, te = H.seq_tols(ref["ell"], w.K)
    tl = np.maximum(1e-4 * np.abs(ref["ell"]), 1e-5)        # eps = log Z + ell - rho - r/beta: ell's bar alone
    g = o.resid.cpu().numpy()
    H.record(test, w.name, seed, "resid (learned log Z)", w.N, np.max(np.abs(g - eps)), H.assert_close_tol(g, eps, tl, "resid"))
    want = O.learned_log_z_grad(eps, w.K, w.N)
    got = dlz.cpu().numpy()
    H.record(test, w.name, seed, "d_log_z", w.B, np.max(np.abs(got - want)),
             H.assert_close_tol(got, want, 2.0 / w.N * tl.reshape(-1, w.K).sum(1), "d_log_z"))
    p0 = o.partial[0].item()
    H.record(test, w.name, seed, "loss", 1, abs(p0 - loss), H.assert_seq_close([p0], [loss], "loss"))
    rows = _row_plan(w, seed, ref["mask"].reshape(-1), [3], 4096)
    n, ma, mr = H.compare_dlogits_rows(d, w, seed, rows, 0, ref["tokens"].reshape(-1), np.repeat(eps, w.T), w.N,
                                       what=f"{test} dlogits", inv_temp=a)
    H.record(test, w.name, seed, "dlogits (group 3 whole + 4096 random rows)", n, ma, mr, tol="1 bf16 ulp")


@pytest.mark.parametrize("name,seed,groups", [("qwen_shard", 1, [0, 5]), ("rhomath", 1, [3, 30]),
                                              ("pythia_fp32", 0, [0, 63])])
def test_deferred_full_size(name, seed, groups):
    """The deferred-scale pass (NEXT 2 (ii)) at full size in the bench's launch configuration: every
    per-sequence value against the oracle, and G = inv_temp (onehot - softmax) — the oracle's
    dlogits_row at c = 1 — on 4096 seeded random valid rows plus every row of two whole groups
    (bf16 G within 1 bf16 ulp, fp32 G within 2e-6; App. A)."""
    w = syn.WORKLOADS[name]
    test = f"deferred_{name}"
    inp = H.device_inputs(w, seed)
    gdt = torch.float32 if w.dtype == "fp32" else torch.bfloat16
    o, _, G = tba.vargrad_fwd_deferred(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"],
                                       inp["log_reward"], w.beta, w.K, float(w.N), g_dtype=gdt, check_status=True)
    torch.cuda.synchronize()
    ref = check_seq_values(test, w, seed, o, 0, w.B, w.N)
    mask_flat = ref["mask"].reshape(-1)
    rows = _row_plan(w, seed, mask_flat, groups, 4096)
    unit = np.full(w.N * w.T, w.N / 2.0)  # eps = N/2 makes the oracle's c = 2 eps / N = 1: dlogits_row = G
    n, ma, mr = H.compare_dlogits_rows(G, w, seed, rows, 0, ref["tokens"].reshape(-1), unit, w.N,
                                       what=f"{test} G, groups {groups} whole + 4096 random rows")
    H.record(test, w.name, seed, f"G (groups {groups} whole + 4096 random rows)", n, ma, mr,
             tol="1 bf16 ulp" if gdt == torch.bfloat16 else "2e-6")
    masked = np.flatnonzero(mask_flat == 0)
    flat = G.view(-1, w.V)
    for i in range(0, len(masked), 4096):                                     # every masked row is +0
        idx = torch.from_numpy(masked[i:i + 4096]).to(G.device)
        assert torch.count_nonzero(flat.index_select(0, idx)).item() == 0
