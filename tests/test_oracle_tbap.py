"""Pins for the TBA' oracle (Eq. 16). CPU only."""
import math

import numpy as np
import pytest

from oracle import tba_oracle as O


def _inst(seed, B=2, K=3, T=4, V=6, p_mask=0.8):
    rng = np.random.default_rng(seed)
    N = B * K
    logits = rng.normal(0, 1.5, size=(N, T, V))
    tokens = rng.integers(0, V, size=(N, T))
    mask = (rng.random((N, T)) < p_mask).astype(np.uint8)
    mask[:, 0] = 1
    ref = rng.normal(-6, 1, N)
    rew = rng.integers(0, 2, N).astype(float)
    return logits, tokens, mask, ref, rew


def _on_policy_gen(logits, tokens, mask):
    """pi_gen = pi_theta: gen log-probs equal the current per-token log-probs."""
    N, T = tokens.shape
    g = np.zeros((N, T))
    for s in range(N):
        for t in range(T):
            if mask[s, t]:
                g[s, t], _ = O.token_logprob(logits[s, t], int(tokens[s, t]))
    return g


def test_beta0_on_policy_is_dr_grpo():  # Dr. GRPO is exactly TBA' at beta = 0
    logits, tokens, mask, ref, rew = _inst(0)
    gen = _on_policy_gen(logits, tokens, mask)
    h = O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.0, 3, "clip", 0.0, 8.0)
    # Eq. 14 written out independently: sg(min(lambda, 8) (r - rbar)) with lambda = 1
    K = 3
    for s in range(len(rew)):
        i = s // K
        rbar = rew[i * K:(i + 1) * K].mean()
        for t in range(tokens.shape[1]):
            want = min(1.0, 8.0) * (rew[s] - rbar) if mask[s, t] else 0.0
            assert abs(h["coef"][s, t] - want) < 1e-12


def test_on_policy_links_eq7_and_eq16():
    """With lambda = 1 and no IS, Eq. 16's bracket is App. A's advantage (A = -beta eps), so
    TBA' dlogits = (beta N / (2 n_tok)) x the VarGrad TB dlogits of Eq. 5."""
    logits, tokens, mask, ref, rew = _inst(1, B=3, K=4, T=3, V=5)
    beta, K = 0.4, 4
    gen = _on_policy_gen(logits, tokens, mask)
    p = O.tbap_head(logits, tokens, mask, gen, ref, rew, beta, K, "none")
    tb = O.vargrad_head(logits, tokens, mask, ref, rew, beta, K)
    np.testing.assert_allclose(p["adv"], -beta * tb["eps"], atol=1e-10)
    np.testing.assert_allclose(p["adv"], O.advantages(tb["ell"], ref, rew, beta, K), atol=1e-12)
    N, ntok = len(rew), int(mask.sum())
    np.testing.assert_allclose(p["dlogits"], beta * N / (2 * ntok) * tb["dlogits"], rtol=1e-9, atol=1e-15)


def test_group_sums_and_shift_invariance():
    logits, tokens, mask, ref, rew = _inst(2, B=2, K=5)
    gen = _on_policy_gen(logits, tokens, mask) + 0.1
    a = O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.05, 5, "clip")
    for i in range(2):
        assert abs(a["adv"][i * 5:(i + 1) * 5].sum()) < 1e-12
    shift = np.repeat([0.7, -1.3], 5)
    b = O.tbap_head(logits, tokens, mask, gen, ref, rew + shift, 0.05, 5, "clip")
    np.testing.assert_allclose(b["adv"], a["adv"], atol=1e-12)
    c = O.tbap_head(logits, tokens, mask, gen, ref + shift, rew, 0.05, 5, "clip")  # ref shift per group
    np.testing.assert_allclose(c["adv"], a["adv"], atol=1e-12)


def test_is_weights_worked_values():
    # CISPO clip (Table 5: lower/upper bound 0/8): ratio 12 -> 8 (S: "sequence ratio 12 with clip_high 8")
    assert O.is_weight(12.0, "clip", 0.0, 8.0) == 8.0
    assert O.is_weight(0.3, "clip", 0.0, 8.0) == 0.3
    assert O.is_weight(0.3, "icepop", 0.5, 2.0) == 0.0 and O.is_weight(3.0, "icepop", 0.5, 2.0) == 0.0
    assert O.is_weight(1.7, "icepop", 0.5, 2.0) == 1.7
    assert O.is_weight(123.0, "none", 0.0, 0.0) == 1.0
    with pytest.raises(ValueError):
        O.is_weight(1.0, "bogus", 0, 1)


def test_icepop_infinite_band_is_unclipped_and_clip_monotone():
    logits, tokens, mask, ref, rew = _inst(3)
    gen = _on_policy_gen(logits, tokens, mask) + np.random.default_rng(3).normal(0, 1.5, tokens.shape)
    a = O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.1, 3, "icepop", 0.0, math.inf)
    b = O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.1, 3, "clip", 0.0, math.inf)
    np.testing.assert_allclose(a["coef"], b["coef"], rtol=0, atol=0)
    c = O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.1, 3, "clip", 0.0, 2.0)
    assert np.all(np.abs(c["coef"]) <= np.abs(b["coef"]) + 1e-15)


def test_finite_differences_with_coefficients_fixed():
    """sg(): the coefficient is a constant; dL'/dz = -(coef/n_tok)(onehot - p) equals central
    differences of L'(z) = -(1/n_tok) sum coef_t lp_t(z) with coef frozen."""
    logits, tokens, mask, ref, rew = _inst(4, B=1, K=2, T=3, V=4)
    gen = _on_policy_gen(logits, tokens, mask) - 0.2
    h = O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.3, 2, "clip")
    coef, n = h["coef"], int(mask.sum())

    def surrogate(lg):
        tot = 0.0
        for s in range(2):
            for t in range(3):
                if mask[s, t]:
                    tot += coef[s, t] * O.token_logprob(lg[s, t], int(tokens[s, t]))[0]
        return -tot / n

    fd = np.zeros_like(logits)
    for idx in np.ndindex(logits.shape):
        lp_, lm_ = logits.copy(), logits.copy()
        lp_[idx] += 1e-5
        lm_[idx] -= 1e-5
        fd[idx] = (surrogate(lp_) - surrogate(lm_)) / 2e-5
    rel = np.max(np.abs(fd - h["dlogits"])) / np.max(np.abs(h["dlogits"]))
    assert rel < 1e-6
    assert abs(h["loss"] - surrogate(logits)) < 1e-14


def test_config_errors():
    logits, tokens, mask, ref, rew = _inst(5)
    gen = np.zeros(tokens.shape)
    with pytest.raises(ValueError):
        O.tbap_head(logits, tokens, mask, gen, ref, rew, -0.1, 3)
    with pytest.raises(ValueError):
        O.tbap_head(logits, tokens, mask, gen, ref, rew, 0.1, 1)


def test_tbap_dlogits_row_finite_differences():
    """tbap_dlogits_row (the expected value of every sampled full-size TBA' row comparison) against
    central differences of the token log-prob it scales: -(coef / n_tok) g d lp / dz."""
    import math
    rng = np.random.default_rng(5)
    for V in (2, 5, 9):
        z = rng.normal(0, 1.5, V)
        y = int(rng.integers(0, V))
        coef, n, g = float(rng.normal()), int(rng.integers(3, 50)), float(rng.normal())
        d = O.tbap_dlogits_row(z, y, coef, n, g)
        h = 1e-6
        for v in range(V):
            zp, zm = z.copy(), z.copy()
            zp[v] += h
            zm[v] -= h
            fd = -(coef / n) * g * (O.token_logprob(zp, y)[0] - O.token_logprob(zm, y)[0]) / (2 * h)
            assert abs(d[v] - fd) <= 1e-8 * max(1.0, abs(fd)), (V, v, d[v], fd)
        assert abs(math.fsum(d)) <= 1e-15
