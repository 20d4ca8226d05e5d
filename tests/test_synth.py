"""The seeded generator (tba_synth): NumPy twin pins. The CUDA twin is checked against it
bit-for-bit in tests/test_gpu_parity.py."""
import numpy as np
import torch

import tba_synth as syn


def test_splitmix64_reference_output():
    # SplitMix64 (Steele, Lea & Flood 2014; Vigna's splitmix64.c) started at state 0:
    # the first output is 0xE220A8397B1DCDAF.
    assert syn.splitmix64_scalar(0, 0) == 0xE220A8397B1DCDAF


def test_vectorised_hash_matches_scalar():
    key = syn.stream_key(7, syn.S_LOGITS)
    idx = np.array([0, 1, 2, 12345, 2 ** 40 + 3], dtype=np.uint64)
    v = syn.hash64(7, syn.S_LOGITS, idx)
    for i, h in zip(idx, v):
        assert int(h) == syn.splitmix64_scalar(key, int(i))


def test_mulhi_exact():
    rng = np.random.default_rng(0)
    h = rng.integers(0, 2 ** 63, size=1000, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    for n in [2, 1000, 50257, 152064, 2 ** 32 - 1]:
        got = syn.mulhi_u64(h, n)
        exp = [(int(x) * n) >> 64 for x in h]
        assert [int(g) for g in got] == exp


def test_bf16_rounding_matches_torch():
    z = syn.logits_rows_f32(0, 4096, np.arange(4))
    a = syn.f32_to_bf16_bits(z)
    b = torch.from_numpy(z).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(a, b)


def test_logits_distribution_and_peak():
    V = 20000
    rows = np.arange(50)
    z = syn.logits_rows_f32(1, V, rows)
    y = syn.raw_tokens(1, V, rows)
    b = syn.peak_of(1, rows)
    body = z.copy()
    body[np.arange(50), y] -= b
    assert np.all(np.abs(body) <= 8.0)
    assert abs(body.mean()) < 0.01 and abs(body.std() - 2.3094) < 0.01   # Irwin-Hall(4) * 2^16 / 2^14
    assert set(np.unique(b)) <= {0.0, 4.0, 8.0, 12.0}
    # values are multiples of 2^-14 (exact in fp32)
    assert np.all(np.mod(body.astype(np.float64) * 2 ** 14, 1.0) == 0.0)


def test_determinism_and_row_independence():
    a = syn.logits_rows(3, 777, [5, 6, 7], "bf16")
    b = syn.logits_rows(3, 777, [7, 6, 5], "bf16")[::-1]
    np.testing.assert_array_equal(a, b)
    c = syn.logits_rows(4, 777, [5, 6, 7], "bf16")
    assert np.mean(a == c) < 0.1


def test_tokens_masks_lengths():
    w = syn.WORKLOADS["rhomath"]
    tok, mask = syn.tokens_and_mask(w, 0)
    L = syn.seq_lengths(w, 0)
    assert tok.shape == (w.N, w.T) and mask.dtype == np.uint8
    assert np.all((L >= 64) & (L <= 512))
    np.testing.assert_array_equal(mask.sum(1), L)
    assert np.all(tok[mask == 0] == -1) and np.all((tok[mask == 1] >= 0) & (tok[mask == 1] < w.V))
    # tokens of a sub-range equal the same sequences of the whole batch
    t2, m2 = syn.tokens_and_mask(w, 0, seq0=40, n=20)
    np.testing.assert_array_equal(t2, tok[40:60])
    np.testing.assert_array_equal(m2, mask[40:60])


def test_rewards_and_ref():
    for name in ["toy", "pythia", "rhomath", "redteam", "qwen"]:
        w = syn.WORKLOADS[name]
        r = syn.log_reward(w, 0)
        ref = syn.ref_logp(w, 0)
        assert r.shape == (w.N,) and ref.shape == (w.N,)
        assert np.all(r.astype(np.float32) == r) and np.all(ref.astype(np.float32) == ref)
        if w.reward == "binary":
            assert set(np.unique(r)) <= {0.0, 1.0}
        if w.reward == "redteam":
            assert np.all(r <= 0) and np.all(r >= -12)
    w = syn.WORKLOADS["qwen"]
    ref = syn.ref_logp(w, 0)
    e_v = 6 - (np.log(w.V) + 2.65)
    assert np.all(np.abs(ref - e_v * w.T) <= 20.0 + 1e-3)


def test_paper_table_presets():
    """Batch shapes of the paper's hyperparameter tables."""
    W = syn.WORKLOADS
    assert (W["gsm8k_t3"].B, W["gsm8k_t3"].K, W["gsm8k_t3"].T) == (7, 20, 512)       # effective batch 140
    assert W["gsm8k_k40"].K == 40 and W["gsm8k_k40"].N <= 140
    assert (W["tldr_t4"].B, W["tldr_t4"].K, W["tldr_t4"].T) == (8, 20, 128)          # effective batch 160
    assert (W["math_t5"].N, W["math_t5"].T, W["math_t5"].beta) == (512, 2048, 0.005)  # 3072 - 1024
    assert W["math_t5_shard"].B * 8 == W["math_t5"].B
    L = syn.seq_lengths(W["math_t5"], 0)
    assert L.min() >= 256 and L.max() <= 2048 and len(L) == 512
    assert np.all(syn.seq_lengths(W["tldr_t4"], 0) == 128)


def test_host_twin_bit_identical_to_numpy():
    """The C host twin (used by the full-size oracle harness) equals the NumPy twin bit for bit,
    bf16 and fp32, on rows spanning small and 64-bit-scale indices and an unaligned vocabulary."""
    rows = np.array([0, 1, 77, 65535, 524287, 2 ** 33 + 5], dtype=np.int64)
    for V in (1000, 50257, 152064):
        for dt in ("bf16", "fp32"):
            a = syn.logits_rows(5, V, rows, dt)
            b = syn.logits_rows_host(5, V, rows, dt)
            assert a.dtype == b.dtype
            np.testing.assert_array_equal(a.view(np.uint16 if dt == "bf16" else np.uint32),
                                          b.view(np.uint16 if dt == "bf16" else np.uint32))
    np.testing.assert_array_equal(syn.logits_rows_f64_host(2, 999, [3, 4], "bf16"),
                                  syn.logits_rows_f64(2, 999, [3, 4], "bf16"))
