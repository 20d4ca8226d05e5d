"""Pins for the fp64 oracle (CPU only). The oracle is never compared with itself: each
check below is fixed by the paper/spec (worked values, closed forms), by mathematics
(invariants, brute force, finite differences) or by an independent library routine."""
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

import tba_synth as syn
from oracle import tba_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))


def _rand_instance(rng, B, K, T, V, p_mask=0.8, scale=2.0):
    N = B * K
    logits = rng.normal(0, scale, size=(N, T, V))
    tokens = rng.integers(0, V, size=(N, T))
    mask = (rng.random((N, T)) < p_mask).astype(np.uint8)
    mask[:, 0] = 1
    ref = rng.normal(-3.0, 1.0, size=N)
    rew = rng.normal(0.0, 1.0, size=N)
    return logits, tokens, mask, ref, rew


# --------------------------------------------------------------------------- worked values
def test_worked_uniform_two_tokens():
    g = GOLD["uniform_v2_two_tokens"]
    logits = np.array(g["logits"])[None]
    ell, ntok, _ = O.seq_logprob(logits, np.array([g["tokens"]]), np.ones((1, 2), np.uint8))
    assert abs(ell[0] - g["seq_logp"]) < 1e-15 and ntok[0] == 2


def test_worked_logits_2_0():
    g = GOLD["logits_2_0_token0"]
    lp, _ = O.token_logprob(np.array(g["logits"][0]), 0)
    assert abs(lp - g["seq_logp"]) < 1e-15


def test_worked_grad_logprob():
    g = GOLD["grad_logprob_uniform_v2"]
    np.testing.assert_allclose(O.grad_logprob_row(np.array(g["logits"]), g["token"]), g["grad"], atol=1e-16)


def _two_sample_instance(g, policy_logits):
    # one group, K=2, each response is a single token (V=2); sequence j emits token j
    logits = np.array([[policy_logits], [policy_logits]], dtype=np.float64)  # [2,1,2]
    tokens = np.array([[g["tokens"][0]], [g["tokens"][1]]])
    mask = np.ones((2, 1), np.uint8)
    return logits, tokens, mask


def test_worked_log_z_loss_and_dlogits():  # S:133; Eqs. 4-5; App. A
    g = GOLD["log_z_r10_uniform"]
    logits, tokens, mask = _two_sample_instance(g, [0.0, 0.0])
    h = O.vargrad_head(logits, tokens, mask, g["ref_logp"], g["log_reward"], g["beta"], g["K"])
    assert abs(h["log_z"][0] - g["log_z"]) < 1e-15
    np.testing.assert_allclose(h["eps"], g["eps"], atol=1e-15)
    assert abs(h["loss"] - g["loss"]) < 1e-15
    np.testing.assert_allclose(h["dlogits"][:, 0, :], g["dlogits_rows"], atol=1e-15)


def test_closed_form_posterior():  # Eq. 2: at pi_theta = pi*, every delta = log Z, L = 0
    g = GOLD["posterior_closed_form"]
    logits, tokens, mask = _two_sample_instance(g, g["policy_logits"])
    h = O.vargrad_head(logits, tokens, mask, g["ref_logp"], g["log_reward"], g["beta"], g["K"])
    assert abs(h["log_z"][0] - g["log_z"]) < 1e-14
    assert abs(h["log_z"][0] - math.log(0.5 * math.e + 0.5)) < 1e-14
    assert h["loss"] < 1e-28
    assert np.max(np.abs(h["dlogits"])) < 1e-14


def test_advantage_worked_example():  # S:152, App. A
    g = GOLD["advantage_example"]
    # choose ell, rho with ell - rho = log_ratio
    ref = np.array([-5.0, -5.0])
    ell = ref + np.array(g["log_ratio"])
    A = O.advantages(ell, ref, g["log_reward"], g["beta"], g["K"])
    np.testing.assert_allclose(A, g["A"], atol=1e-15)
    loss, _, eps = O.vargrad_tb_loss(ell, ref, g["log_reward"], g["beta"], g["K"])
    np.testing.assert_allclose(eps, g["eps"], atol=1e-14)
    assert abs(loss - g["loss"]) < 1e-15


# --------------------------------------------------------------------------- a1 invariants
@pytest.mark.parametrize("V", [2, 1000, 50257, 152064])
def test_softmax_rows_sum_to_one(V):  # north_star / S:75: within 1e-12
    rows = np.arange(3) + 7
    z = syn.logits_rows_f64(0, V, rows, "bf16")
    for r in z:
        lp, _ = O.log_softmax_row(r)
        assert abs(math.fsum(np.exp(lp)) - 1.0) < 1e-12


def test_softmax_row_sum_extreme():
    z = np.concatenate([np.full(100000, -30.0), [25.0], np.full(52064, 0.0)])
    lp, _ = O.log_softmax_row(z)
    assert abs(math.fsum(np.exp(lp)) - 1.0) < 1e-12


@pytest.mark.parametrize("c", [2.0 ** 5, -(2.0 ** 7), 2.0 ** -3])
def test_shift_invariance(c):  # within 1e-9 (power-of-two shift keeps bf16 values exact)
    z = syn.logits_rows_f64(3, 5000, [11], "bf16")[0]
    a, _ = O.log_softmax_row(z)
    b, _ = O.log_softmax_row(z + c)
    assert np.max(np.abs(a - b)) < 1e-9


def test_against_scipy_logsumexp():  # independent library routine
    z = syn.logits_rows_f64(5, 32000, [1, 2, 3], "bf16")
    for r in z:
        lp, lse = O.log_softmax_row(r)
        assert abs(lse - scipy.special.logsumexp(r)) < 1e-12
        np.testing.assert_allclose(lp, scipy.special.log_softmax(r), atol=1e-12, rtol=0)
        t = torch.from_numpy(r)
        np.testing.assert_allclose(lp, torch.log_softmax(t, 0).numpy(), atol=1e-12, rtol=0)


def test_neg_inf_entries_and_token_range():
    z = np.array([-np.inf, -np.inf, 1.0, 0.0])
    lp, _ = O.log_softmax_row(z)
    assert lp[0] == -np.inf and abs(lp[2] - (1 - math.log(math.e + 1))) < 1e-15
    with pytest.raises(ValueError):
        O.token_logprob(z, 4)
    with pytest.raises(ValueError):
        O.token_logprob(z, -1)


# --------------------------------------------------------------------------- a2 brute force
def test_seq_logprob_brute_force_product():
    rng = np.random.default_rng(1)
    logits, tokens, mask, _, _ = _rand_instance(rng, 2, 3, 4, 5, scale=1.0)
    ell, ntok, _ = O.seq_logprob(logits, tokens, mask)
    for s in range(len(ell)):
        prod = 1.0
        for t in range(4):
            if mask[s, t]:
                e = np.exp(logits[s, t])          # no max subtraction: plain definition
                prod *= e[tokens[s, t]] / e.sum()
        assert abs(math.exp(ell[s]) - prod) < 1e-14 * max(1.0, prod)
        assert ntok[s] == int(mask[s].sum())


def test_row_terms_and_sequence_sums_brute_force():
    """token_logprob_rows + sequence_sums (what the full-size harness calls on regenerated rows)
    against the plain product of probabilities, row by row, with no reference to seq_logprob."""
    rng = np.random.default_rng(11)
    logits, tokens, mask, _, _ = _rand_instance(rng, 2, 2, 5, 6, scale=1.5)
    N, T, V = logits.shape
    valid = np.flatnonzero(mask.reshape(-1))
    lp_v, lse_v = O.token_logprob_rows(logits.reshape(N * T, V)[valid], tokens.reshape(-1)[valid])
    for i, r in enumerate(valid):
        e = np.exp(logits.reshape(N * T, V)[r])
        assert abs(math.exp(lp_v[i]) - e[tokens.reshape(-1)[r]] / e.sum()) < 1e-15
        assert abs(math.exp(lse_v[i]) - e.sum()) < 1e-13 * e.sum()
    lp = np.full((N, T), np.nan)                  # entries at masked positions must be ignored
    lp.reshape(-1)[valid] = lp_v
    ell, ntok = O.sequence_sums(lp, mask)
    for s in range(N):
        prod = 1.0
        for t in range(T):
            if mask[s, t]:
                e = np.exp(logits[s, t])
                prod *= e[tokens[s, t]] / e.sum()
        assert abs(math.exp(ell[s]) - prod) < 1e-14 * max(1.0, prod)
        assert ntok[s] == int(mask[s].sum())


def test_masked_positions_ignored():
    rng = np.random.default_rng(2)
    logits, tokens, mask, _, _ = _rand_instance(rng, 1, 2, 6, 7)
    t2 = tokens.copy()
    t2[mask == 0] = -1                          # garbage tokens where masked
    l2 = logits.copy()
    l2[mask == 0] = np.nan                      # garbage logits where masked
    a = O.seq_logprob(logits, tokens, mask)[0]
    b = O.seq_logprob(l2, t2, mask)[0]
    np.testing.assert_array_equal(a, b)


def test_empty_sequence():
    logits = np.zeros((2, 3, 4))
    mask = np.array([[0, 0, 0], [1, 1, 0]], np.uint8)
    ell, ntok, _ = O.seq_logprob(logits, np.zeros((2, 3), int), mask)
    assert ell[0] == 0.0 and ntok[0] == 0 and ntok[1] == 2


# --------------------------------------------------------------------------- a3 closed forms / invariants
def test_loss_is_mean_group_variance():
    rng = np.random.default_rng(3)
    B, K = 5, 4
    ell, ref, rew = rng.normal(-50, 5, B * K), rng.normal(-50, 5, B * K), rng.normal(0, 1, B * K)
    beta = 0.3
    loss, logz, eps = O.vargrad_tb_loss(ell, ref, rew, beta, K)
    delta = ref - ell + rew / beta
    var = np.mean([np.var(delta[i * K:(i + 1) * K]) for i in range(B)])  # population variance
    assert abs(loss - var) < 1e-12 * max(1, var)
    for i in range(B):
        assert abs(math.fsum(eps[i * K:(i + 1) * K])) < 1e-11   # S:148 sum_j eps = 0


def test_loss_zero_iff_delta_constant_and_shift_invariant():
    rng = np.random.default_rng(4)
    B, K, beta = 3, 5, 0.7
    ref = rng.normal(-20, 3, B * K)
    c = np.repeat(rng.normal(0, 10, B), K)
    rew = rng.normal(0, 1, B * K)
    ell = ref + rew / beta - c               # delta = c_i constant per group
    loss, _, _ = O.vargrad_tb_loss(ell, ref, rew, beta, K)
    assert loss < 1e-24
    ell2 = ell + rng.normal(0, 0.1, B * K)
    l2, _, _ = O.vargrad_tb_loss(ell2, ref, rew, beta, K)
    assert l2 > 1e-6
    shift = np.repeat(rng.normal(0, 3, B), K)  # per-group reward shift
    l3, _, eps3 = O.vargrad_tb_loss(ell2, ref, rew + beta * shift, beta, K)
    assert abs(l3 - l2) < 1e-12 and l3 >= 0


def test_advantage_identity():  # App. A: A = -beta * eps, independent formulas
    rng = np.random.default_rng(5)
    B, K, beta = 4, 6, 0.05
    ell, ref, rew = rng.normal(-300, 20, B * K), rng.normal(-300, 20, B * K), rng.integers(0, 2, B * K).astype(float)
    _, _, eps = O.vargrad_tb_loss(ell, ref, rew, beta, K)
    A = O.advantages(ell, ref, rew, beta, K)
    np.testing.assert_allclose(A, -beta * eps, atol=1e-10)
    for i in range(B):
        assert abs(A[i * K:(i + 1) * K].sum()) < 1e-9


def test_config_errors():
    with pytest.raises(ValueError):
        O.vargrad_tb_loss([0.0, 1.0], [0.0, 0.0], [0.0, 0.0], 0.0, 2)
    with pytest.raises(ValueError):
        O.vargrad_tb_loss([0.0, 1.0], [0.0, 0.0], [0.0, 0.0], float("nan"), 2)
    with pytest.raises(ValueError):
        O.vargrad_tb_loss([0.0], [0.0], [0.0], 1.0, 1)
    with pytest.raises(ValueError):
        O.vargrad_tb_loss([0.0] * 5, [0.0] * 5, [0.0] * 5, 1.0, 2)


# --------------------------------------------------------------------------- a5 finite differences
@pytest.mark.parametrize("K", [2, 3, 4])
def test_dlogits_finite_differences(K):  # north_star / S:160: relative error <= 1e-6
    rng = np.random.default_rng(10 + K)
    B, T, V, beta = 2, 3, 4, 0.7
    logits, tokens, mask, ref, rew = _rand_instance(rng, B, K, T, V)
    h = O.vargrad_head(logits, tokens, mask, ref, rew, beta, K)
    an = h["dlogits"]

    def loss_of(lg):
        return O.vargrad_head(lg, tokens, mask, ref, rew, beta, K, want_grad=False)["loss"]

    fd = np.zeros_like(logits)
    step = 1e-5
    for idx in np.ndindex(logits.shape):
        lp = logits.copy(); lp[idx] += step
        lm = logits.copy(); lm[idx] -= step
        fd[idx] = (loss_of(lp) - loss_of(lm)) / (2 * step)
    rel = np.max(np.abs(fd - an)) / np.max(np.abs(an))
    assert rel < 1e-6, rel


def test_grad_token_entry_confident_closed_form():
    """The token's entry 1 - p_y of a confident row against its closed form 2 / (e^40 + 2) for
    z = (40, 0, 0), y = 0 (8.5e-18: fp64's 1 - p_y would cancel to 0); the other entries -p_v."""
    g = O.grad_logprob_row(np.array([40.0, 0.0, 0.0]), 0)
    assert abs(g[0] - 2.0 / (math.exp(40.0) + 2.0)) <= 1e-13 * g[0]
    np.testing.assert_allclose(g[1:], -1.0 / (math.exp(40.0) + 2.0), rtol=1e-13)
    assert abs(g.sum()) <= 1e-30


def test_dlogits_row_pins():
    """dlogits_row (the expected value of every sampled full-size row comparison): (i) central
    finite differences of the token log-prob it scales, times 2 eps g / N (App. A);
    (ii) the S:133 worked rows (-0.25, +0.25); (iii) equal to the FD-pinned ``dlogits`` at
    (s, t) on random instances with grad_out != 1 and N_global != N."""
    rng = np.random.default_rng(21)
    for V in (2, 3, 7):
        z = rng.normal(0, 1.5, V)
        y = int(rng.integers(0, V))
        eps, n, g = float(rng.normal()), int(rng.integers(4, 40)), float(rng.normal())
        d = O.dlogits_row(z, y, eps, n, g)
        h = 1e-6
        for v in range(V):
            zp, zm = z.copy(), z.copy()
            zp[v] += h
            zm[v] -= h
            fd = (O.token_logprob(zp, y)[0] - O.token_logprob(zm, y)[0]) / (2 * h) * 2 * eps * g / n
            assert abs(d[v] - fd) <= 1e-8 * max(1.0, abs(fd))
    gold = GOLD["log_z_r10_uniform"]
    for j in range(2):
        row = O.dlogits_row(np.zeros(2), gold["tokens"][j], gold["eps"][j], 2)
        np.testing.assert_allclose(row, gold["dlogits_rows"][j], atol=1e-15)
    logits, tokens, mask, ref, rew = _rand_instance(rng, 2, 3, 4, 9)
    _, _, eps = O.vargrad_tb_loss(O.seq_logprob(logits, tokens, mask)[0], ref, rew, 0.5, 3, n_global=20)
    full = O.dlogits(logits, tokens, mask, eps, 20, grad_out=-1.75)
    for s in range(6):
        for t in range(4):
            if mask[s, t]:
                np.testing.assert_allclose(O.dlogits_row(logits[s, t], int(tokens[s, t]), eps[s], 20, -1.75),
                                           full[s, t], rtol=0, atol=1e-16)


def test_dlogits_rows_sum_zero_and_masked_zero():
    rng = np.random.default_rng(20)
    logits, tokens, mask, ref, rew = _rand_instance(rng, 3, 4, 5, 9, p_mask=0.6)
    h = O.vargrad_head(logits, tokens, mask, ref, rew, 0.2, 4, grad_out=1.7)
    d = h["dlogits"]
    assert np.max(np.abs(d.sum(-1))) < 1e-14
    assert np.all(d[mask == 0] == 0.0)


def test_dlogits_grad_out_and_normaliser_linear():
    rng = np.random.default_rng(21)
    logits, tokens, mask, ref, rew = _rand_instance(rng, 2, 2, 3, 5)
    a = O.vargrad_head(logits, tokens, mask, ref, rew, 0.5, 2)["dlogits"]
    b = O.vargrad_head(logits, tokens, mask, ref, rew, 0.5, 2, n_global=40, grad_out=3.0)["dlogits"]
    np.testing.assert_allclose(b, a * 3.0 * 4 / 40, rtol=1e-14, atol=1e-18)


# --------------------------------------------------------------------------- a4 sharding
def test_shard_partials_sum_to_unsharded():
    rng = np.random.default_rng(30)
    B, K, beta = 6, 3, 0.4
    logits, tokens, mask, ref, rew = _rand_instance(rng, B, K, 3, 6)
    full = O.vargrad_head(logits, tokens, mask, ref, rew, beta, K, want_grad=True)
    N = B * K
    parts, grads = [], []
    for g0, g1 in [(0, 2), (2, 3), (3, 6), (6, 6)]:
        sl = slice(g0 * K, g1 * K)
        if g1 == g0:
            parts.append(np.zeros(3))
            continue
        h = O.vargrad_head(logits[sl], tokens[sl], mask[sl], ref[sl], rew[sl], beta, K, n_global=N)
        parts.append(h["partial"])
        grads.append(h["dlogits"])
    tot = np.sum(parts, axis=0)
    assert abs(tot[0] - full["loss"]) < 1e-13 and tot[1] == N and tot[2] == B
    np.testing.assert_allclose(np.concatenate(grads), full["dlogits"], rtol=1e-13, atol=1e-18)


# --------------------------------------------------------------------------- bf16 rounding
def test_round_bf16_against_torch():
    rng = np.random.default_rng(40)
    x32 = np.concatenate([rng.normal(0, 1, 20000), rng.normal(0, 1e-3, 2000), rng.normal(0, 1e-38, 200),
                          [1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 2 ** -130, 0.0]]).astype(np.float32)
    ref = torch.from_numpy(x32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(O.round_bf16(x32.astype(np.float64)), ref)
    assert O.round_bf16(np.array([1 + 2 ** -8]))[0] == 1.0          # tie -> even
    assert O.round_bf16(np.array([1 + 3 * 2 ** -8]))[0] == 1 + 2 ** -6
    u = O.bf16_ulp(np.array([1.0, 1.5, 2.0 ** -130, 0.0]))
    np.testing.assert_array_equal(u, [2 ** -7, 2 ** -7, 2 ** -133, 2 ** -133])
