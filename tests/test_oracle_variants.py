"""Pins for the TB head variants: learned log Z (Eq. 3) and the inverse
temperature. CPU only."""
import math

import numpy as np

from oracle import tba_oracle as O


def _inst(seed, B=2, K=3, T=3, V=5):
    rng = np.random.default_rng(seed)
    N = B * K
    return (rng.normal(0, 1.5, (N, T, V)), rng.integers(0, V, (N, T)),
            (rng.random((N, T)) < 0.8).astype(np.uint8), rng.normal(-4, 1, N), rng.normal(0, 1, N))


def test_learned_z_at_vargrad_estimate_equals_vargrad():
    """The Eq. 4 estimate minimises Eq. 3's batch loss over log Z: plugging it in reproduces
    Eq. 5 exactly and the log Z gradient vanishes."""
    logits, tokens, mask, ref, rew = _inst(0)
    v = O.vargrad_head(logits, tokens, mask, ref, rew, 0.5, 3)
    l = O.vargrad_head(logits, tokens, mask, ref, rew, 0.5, 3, log_z=v["log_z"])
    np.testing.assert_allclose(l["eps"], v["eps"], atol=1e-13)
    assert abs(l["loss"] - v["loss"]) < 1e-13
    np.testing.assert_allclose(l["d_log_z"], 0.0, atol=1e-12)
    np.testing.assert_allclose(l["dlogits"], v["dlogits"], atol=1e-14)


def test_learned_z_posterior_closed_form():  # Eq. 2/3: log Z = log(0.5e + 0.5), pi = pi* -> L = 0
    logits = np.array([[[1.0, 0.0]], [[1.0, 0.0]]])
    tokens = np.array([[0], [1]])
    mask = np.ones((2, 1), np.uint8)
    ref = np.log([0.5, 0.5])
    h = O.vargrad_head(logits, tokens, mask, ref, [1.0, 0.0], 1.0, 2, log_z=[math.log(0.5 * math.e + 0.5)])
    assert h["loss"] < 1e-28 and abs(h["d_log_z"][0]) < 1e-14


def test_learned_z_finite_differences():
    logits, tokens, mask, ref, rew = _inst(1, B=2, K=2, T=2, V=3)
    lz = np.array([0.3, -1.2])
    h = O.vargrad_head(logits, tokens, mask, ref, rew, 0.7, 2, log_z=lz)

    def loss(lg, z):
        return O.vargrad_head(lg, tokens, mask, ref, rew, 0.7, 2, log_z=z, want_grad=False)["loss"]

    for i in range(2):
        zp, zm = lz.copy(), lz.copy()
        zp[i] += 1e-6
        zm[i] -= 1e-6
        assert abs((loss(logits, zp) - loss(logits, zm)) / 2e-6 - h["d_log_z"][i]) < 1e-6 * max(1, abs(h["d_log_z"][i]))
    fd = np.zeros_like(logits)
    for idx in np.ndindex(logits.shape):
        a, b = logits.copy(), logits.copy()
        a[idx] += 1e-5
        b[idx] -= 1e-5
        fd[idx] = (loss(a, lz) - loss(b, lz)) / 2e-5
    assert np.max(np.abs(fd - h["dlogits"])) / np.max(np.abs(h["dlogits"])) < 1e-6


def test_inverse_temperature_scaling_identity_and_fd():
    logits, tokens, mask, ref, rew = _inst(2, B=1, K=3, T=2, V=4)
    a = 1 / 0.7
    h = O.vargrad_head(logits, tokens, mask, ref, rew, 0.3, 3, inv_temp=a)
    g = O.vargrad_head(logits * a, tokens, mask, ref, rew, 0.3, 3)
    np.testing.assert_allclose(h["ell"], g["ell"], atol=1e-13)
    np.testing.assert_allclose(h["dlogits"], a * g["dlogits"], atol=1e-13)
    one = O.vargrad_head(logits, tokens, mask, ref, rew, 0.3, 3, inv_temp=1.0)
    base = O.vargrad_head(logits, tokens, mask, ref, rew, 0.3, 3)
    np.testing.assert_array_equal(one["dlogits"], base["dlogits"])

    def loss(lg):
        return O.vargrad_head(lg, tokens, mask, ref, rew, 0.3, 3, inv_temp=a, want_grad=False)["loss"]

    fd = np.zeros_like(logits)
    for idx in np.ndindex(logits.shape):
        p, m = logits.copy(), logits.copy()
        p[idx] += 1e-5
        m[idx] -= 1e-5
        fd[idx] = (loss(p) - loss(m)) / 2e-5
    assert np.max(np.abs(fd - h["dlogits"])) / np.max(np.abs(h["dlogits"])) < 1e-6


def test_row_functions_with_temperature_equal_the_head():
    """token_logprob_rows / dlogits_row with inv_temp (what the full-size harness calls) equal the
    per-row entries of vargrad_head(inv_temp=...) (itself pinned by FD and the scaling identity)."""
    rng = np.random.default_rng(9)
    N, T, V, K = 4, 3, 11, 2
    z = rng.normal(0, 2, (N, T, V))
    tok = rng.integers(0, V, (N, T))
    mask = np.ones((N, T), np.uint8)
    ref, rew = rng.normal(-5, 1, N), rng.normal(0, 1, N)
    a = 1 / 0.7
    h = O.vargrad_head(z, tok, mask, ref, rew, 0.4, K, inv_temp=a, grad_out=1.3)
    lp, _ = O.token_logprob_rows(z.reshape(N * T, V), tok.reshape(-1), inv_temp=a)
    ell, _ = O.sequence_sums(lp.reshape(N, T), mask)
    np.testing.assert_allclose(ell, h["ell"], rtol=0, atol=1e-13)
    for s in range(N):
        for t in range(T):
            np.testing.assert_allclose(O.dlogits_row(z[s, t], int(tok[s, t]), h["eps"][s], N, 1.3, inv_temp=a),
                                       h["dlogits"][s, t], rtol=0, atol=1e-15)
