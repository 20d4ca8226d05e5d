"""Pins of the LM-head-fused oracle (NEXT 3): z = W h followed by the pinned log-softmax."""
import math

import numpy as np
import pytest

import tba_synth as syn
from oracle import tba_oracle as O


def _brute(h, W, y):
    # triple loop, pure Python floats: z_v = sum_i h_i W_vi; log softmax by definition
    z = [sum(float(h[i]) * float(W[v][i]) for i in range(len(h))) for v in range(len(W))]
    return z[y] - math.log(sum(math.exp(zv) for zv in z))


def test_brute_force_tiny():
    rng = np.random.default_rng(0)
    H = rng.normal(size=(5, 3))
    W = rng.normal(size=(4, 3))
    y = np.array([0, 3, 1, 2, 3])
    got = O.lmhead_token_logprob(H, W, y)
    for r in range(5):
        assert abs(got[r] - _brute(H[r], W, y[r])) < 1e-13


def test_logits_are_dot_products():
    rng = np.random.default_rng(1)
    H, W = rng.normal(size=(3, 7)), rng.normal(size=(5, 7))
    z = O.lmhead_logits(H, W)
    for r in range(3):
        for v in range(5):
            assert abs(z[r, v] - math.fsum(H[r, i] * W[v, i] for i in range(7))) < 1e-13


def test_equal_weight_rows_give_uniform():
    rng = np.random.default_rng(2)
    V, d = 37, 16
    W = np.tile(rng.normal(size=(1, d)), (V, 1))
    H = rng.normal(size=(6, d)) * 5
    lp = O.lmhead_token_logprob(H, W, rng.integers(0, V, 6))
    np.testing.assert_allclose(lp, -math.log(V), rtol=0, atol=1e-13)


def test_one_hot_weight_rows_closed_form():
    # W_v = c e_{v mod d}: z_v = c h_{v mod d}
    V, d, c = 10, 4, 0.75
    W = np.zeros((V, d))
    W[np.arange(V), np.arange(V) % d] = c
    h = np.array([0.3, -1.2, 2.0, 0.1])
    z = c * h[np.arange(V) % d]
    for y in range(V):
        want = z[y] - math.log(sum(math.exp(t) for t in z))
        assert abs(O.lmhead_token_logprob(h[None], W, [y])[0] - want) < 1e-13


def test_common_shift_of_weight_rows_is_invariant():
    rng = np.random.default_rng(3)
    H, W, u = rng.normal(size=(4, 8)), rng.normal(size=(30, 8)), rng.normal(size=8)
    y = rng.integers(0, 30, 4)
    np.testing.assert_allclose(O.lmhead_token_logprob(H, W + u, y), O.lmhead_token_logprob(H, W, y),
                               rtol=0, atol=1e-12)


def test_temperature_is_weight_scaling_and_chunked_callable():
    rng = np.random.default_rng(4)
    H, W = rng.normal(size=(3, 8)), rng.normal(size=(50, 8))
    y = rng.integers(0, 50, 3)
    a = O.lmhead_token_logprob(H, W, y, inv_temp=1 / 0.7)
    np.testing.assert_allclose(a, O.lmhead_token_logprob(H, W / 0.7, y), rtol=0, atol=1e-12)

    def gen(v0, v1):
        return W[v0:v1]
    gen.vocab = 50
    np.testing.assert_allclose(O.lmhead_token_logprob(H, gen, y, inv_temp=1 / 0.7, chunk=7), a, rtol=0, atol=1e-13)


def test_seq_logprob_sums_tokens():
    rng = np.random.default_rng(5)
    N, T, d, V = 2, 3, 4, 9
    H, W = rng.normal(size=(N, T, d)), rng.normal(size=(V, d))
    tok = rng.integers(0, V, (N, T))
    mask = np.array([[1, 1, 0], [1, 0, 0]], np.uint8)
    ell, n = O.lmhead_seq_logprob(H, W, tok, mask)
    assert list(n) == [2, 1]
    assert abs(ell[0] - (_brute(H[0, 0], W, tok[0, 0]) + _brute(H[0, 1], W, tok[0, 1]))) < 1e-12
    assert abs(ell[1] - _brute(H[1, 0], W, tok[1, 0])) < 1e-12


@pytest.mark.parametrize("kind", ["normal", "lattice"])
def test_generator_lmhead_inputs(kind):
    h = syn.bf16_bits_to_f64(syn.hidden_rows(0, 64, np.arange(8), kind))
    w = syn.bf16_bits_to_f64(syn.weight_rows(0, 64, np.arange(100), kind))
    assert h.shape == (8, 64) and w.shape == (100, 64)
    if kind == "lattice":
        assert set(np.unique(h * 4)).issubset({-2, -1, 0, 1, 2})
        z = O.lmhead_logits(h, w)
        assert np.all(z * 16 == np.round(z * 16))  # multiples of 1/16: exact in fp32 at any order
    else:
        assert 0.9 < h.std() < 1.4
        # rows are counter-indexed: a sub-range equals the matching rows of a larger call
        assert np.array_equal(syn.weight_rows(0, 64, np.arange(40, 60), kind), syn.weight_rows(0, 64, np.arange(100), kind)[40:60])


# ---- backward through the LM head (lmhead_grads): pinned by finite differences of the loss
def _tiny_lm_case(seed, inv_temp=1.0, learned=False):
    rng = np.random.default_rng(seed)
    B, K, T, d, V = 2, 2, 3, 5, 7
    N = B * K
    H, W = rng.normal(size=(N, T, d)), rng.normal(size=(V, d))
    tok = rng.integers(0, V, (N, T))
    mask = np.array([[1, 1, 1], [1, 1, 0], [1, 0, 0], [1, 1, 1]], np.uint8)
    ref, rew = rng.normal(size=N) * 2, rng.uniform(0, 1, N)
    log_z = rng.normal(size=B) if learned else None

    def loss(Hx, Wx):
        z = O.lmhead_logits(Hx.reshape(N * T, d), Wx).reshape(N, T, V)
        return O.vargrad_head(z, tok, mask, ref, rew, 0.7, K, want_grad=False, inv_temp=inv_temp,
                              log_z=log_z)["loss"]

    z = O.lmhead_logits(H.reshape(N * T, d), W).reshape(N, T, V)
    r = O.vargrad_head(z, tok, mask, ref, rew, 0.7, K, inv_temp=inv_temp, log_z=log_z)
    dH, dW = O.lmhead_grads(H.reshape(N * T, d), W, r["dlogits"].reshape(N * T, V))
    return H, W, loss, dH.reshape(N, T, d), dW, mask


@pytest.mark.parametrize("inv_temp,learned", [(1.0, False), (1 / 0.7, False), (1.0, True)])
def test_lmhead_grads_match_central_differences(inv_temp, learned):
    H, W, loss, dH, dW, mask = _tiny_lm_case(7, inv_temp, learned)
    h = 1e-6
    for arr, g in ((H, dH), (W, dW)):
        fd = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = arr[i]
            arr[i] = old + h
            lp = loss(H, W)
            arr[i] = old - h
            lm = loss(H, W)
            arr[i] = old
            fd[i] = (lp - lm) / (2 * h)
        err = np.max(np.abs(fd - g)) / max(np.max(np.abs(g)), 1e-12)
        assert err < 1e-6, err
    # masked rows get no gradient
    assert np.all(dH[mask == 0] == 0.0)


def test_lmhead_dw_vocab_sum_is_zero_and_equal_rows_give_zero_dh():
    # sum_v (onehot - softmax)_v = 0 for every row, so sum_v dW_v = sum_r 0 * h_r = 0
    H, W, _, dH, dW, _ = _tiny_lm_case(8)
    np.testing.assert_allclose(dW.sum(axis=0), 0.0, atol=1e-13)
    # equal weight rows: dH_r = sum_v dz_rv W_0 = 0
    rng = np.random.default_rng(9)
    Wc = np.tile(rng.normal(size=(1, 6)), (11, 1))
    Hc = rng.normal(size=(5, 6))
    dz = np.stack([O.grad_logprob_row(O.lmhead_logits(Hc[r:r + 1], Wc)[0], r) for r in range(5)])
    dHc, _ = O.lmhead_grads(Hc, Wc, dz)
    np.testing.assert_allclose(dHc, 0.0, atol=1e-14)
