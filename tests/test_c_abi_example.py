"""The C ABI is usable from plain C: examples/c_abi_example.c builds here (CPU) and, on a GPU,
its printed loss / per-sequence log-probs match the fp64 oracle on the same inputs."""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import tba_oracle as O

from . import _harness as H


def _inputs():
    N, T, V = 6, 4, 257
    st = 88172645463325252
    M = (1 << 64) - 1

    def nxt(x):
        x ^= (x << 13) & M
        x ^= x >> 7
        x ^= (x << 17) & M
        return x

    logits = np.empty(N * T * V, np.float32)
    for i in range(N * T * V):
        st = nxt(st)
        logits[i] = np.float32((st >> 11) / 9007199254740992.0 * 8.0 - 4.0)
    tok = np.empty(N * T, np.int64)
    mask = np.empty(N * T, np.uint8)
    for i in range(N * T):
        st = nxt(st)
        tok[i] = st % V
        mask[i] = 1 if (i % T) < T - (i // T) % 2 else 0
    ref = np.array([-20.0 + s for s in range(N)])
    rew = np.array([float(s % 2) for s in range(N)])
    D = 64
    vals = np.empty(N * T * D + V * D)
    for i in range(len(vals)):
        st = nxt(st)
        vals[i] = (int(st % 5) - 2) * 0.25
    hid = vals[:N * T * D].reshape(N * T, D)
    w = vals[N * T * D:].reshape(V, D)
    return (logits.reshape(N, T, V).astype(np.float64), tok.reshape(N, T), mask.reshape(N, T), ref, rew,
            hid, w)


def test_c_example_compiles():
    from paper_2503_18929_b200 import _build
    assert _build.build_c_example()


@pytest.mark.gpu
def test_c_example_runs_and_matches_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_18929_b200 import _build
    exe = _build.build_c_example()
    import tempfile
    dump = os.path.join(tempfile.mkdtemp(), "dlogits.f32")
    out = subprocess.run([exe, dump], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    logits, tok, mask, ref, rew, hid, w = _inputs()
    r = O.vargrad_head(logits, tok, mask, ref, rew, 0.5, 3)
    m = re.search(r"status 0 loss (\S+) n_seq 6 n_groups 2", out.stdout)
    assert m, out.stdout
    assert abs(float(m.group(1)) - r["loss"]) <= 1e-4 * abs(r["loss"])
    got = [float(x) for x in re.findall(r"seq \d+ logp (\S+) ntok", out.stdout)]
    np.testing.assert_allclose(got, r["ell"], rtol=1e-6)
    cs = float(re.search(r"dlogits_abs_sum (\S+)", out.stdout).group(1))
    assert abs(cs - np.abs(r["dlogits"]).sum()) <= 1e-5 * np.abs(r["dlogits"]).sum()
    # every element of the fp32 dlogits the C program wrote, against the oracle (R9 bar)
    d = np.fromfile(dump, dtype=np.float32).astype(np.float64).reshape(r["dlogits"].shape)
    for s in range(d.shape[0]):
        c = 2.0 * r["eps"][s] / d.shape[0]
        for t in range(d.shape[1]):
            H.assert_dlogits_close(d[s, t], r["dlogits"][s, t], c, "fp32", f"C example s={s} t={t}")
    # the LM-head-fused forward from the lattice hidden states (exact logits)
    ell, _ = O.lmhead_seq_logprob(hid.reshape(6, 4, 64), w, tok, mask)
    got = [float(x) for x in re.findall(r"lmhead seq \d+ logp (\S+)", out.stdout)]
    np.testing.assert_allclose(got, ell, rtol=0, atol=1e-5)
    # the one-call LM-head training step: loss and the gradient sums
    z = O.lmhead_logits(hid, w).reshape(6, 4, 257)
    rl = O.vargrad_head(z, tok, mask, ref, rew, 0.5, 3)
    dH, dW = O.lmhead_grads(hid, w, rl["dlogits"].reshape(24, 257))
    m = re.search(r"lmhead loss (\S+) dhidden_abs_sum (\S+) dweight_abs_sum (\S+)", out.stdout)
    assert m, out.stdout
    assert abs(float(m.group(1)) - rl["loss"]) <= 1e-4 * abs(rl["loss"])
    # |sum|x| - sum|x_ref|| <= sum |x - x_ref| <= the per-element bound of DESIGN.md R21, summed
    AZ = np.abs(rl["dlogits"].reshape(24, 257))
    assert abs(float(m.group(2)) - np.abs(dH).sum()) <= (2.0 ** -8 + 4 * 257 ** 0.5 * 2.0 ** -24) * (AZ @ np.abs(w)).sum()
    assert abs(float(m.group(3)) - np.abs(dW).sum()) <= (2.0 ** -8 + 4 * 24 ** 0.5 * 2.0 ** -24) * (AZ.T @ np.abs(hid)).sum()
