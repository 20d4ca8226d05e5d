"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Per-sequence values are compared with the fp64 oracle on every sequence the oracle can
afford (all of Pythia and red-teaming; sampled whole groups of RhoMath and of the Qwen
per-GPU shard), dlogits on seeded samples of rows; properties that hold at any size
(loss = sum eps^2 / N, sum_v dlogits = 0, masked rows zero, group permutation and reward
shift metamorphics, bitwise determinism) are checked on the full outputs."""
import dataclasses

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


def check_groups(w, seed, inp, o, d, groups, n_rows_sample=48):
    """Oracle on whole groups `groups` (per-sequence values) + sampled rows of dlogits."""
    K, T = w.K, w.T
    N = inp["tokens"].shape[0]
    sl, nt = o.seq_logp.cpu().numpy(), o.n_tokens.cpu().numpy()
    lz, eps = o.log_z.cpu().numpy(), o.resid.cpu().numpy()
    rng = np.random.default_rng(seed + 100)
    for g in groups:
        ref = H.oracle_seq_values(w, seed, g, 1)
        s = slice(g * K, (g + 1) * K)
        H.assert_seq_close(sl[s], ref["ell"], f"seq_logp group {g}")
        np.testing.assert_array_equal(nt[s], ref["n_tok"])
        loss_g, logz_g, eps_g = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, K,
                                                  n_global=N)
        H.assert_seq_close(lz[g:g + 1], logz_g, f"log_z group {g}")
        H.assert_seq_close(eps[s], eps_g, f"resid group {g}")
        # sampled valid rows of this group: oracle dlogits row vs GPU row
        mask = ref["mask"]
        valid = np.flatnonzero(mask.reshape(-1))
        pick = rng.choice(valid, size=min(n_rows_sample, len(valid)), replace=False)
        rows_global = g * K * T + pick
        z = syn.logits_rows_f64(seed, w.V, rows_global, w.dtype)
        for i, r in enumerate(pick):
            sj, t = divmod(int(r), T)
            y = int(ref["tokens"][sj, t])
            want = O.dlogits_row(z[i], y, eps_g[sj], N)
            got = d[g * K + sj, t].float().cpu().numpy().astype(np.float64)
            H.assert_dlogits_close(got, want, 2 * eps_g[sj] / N, w.dtype, f"g={g} s={sj} t={t}")


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
    rows = rng.choice(N * w.T, size=n_rows, replace=False)
    for r in rows:
        row = flat[r].float()
        if mask.reshape(-1)[r]:
            c = abs(2 * eps[r // w.T] / N)
            assert abs(row.double().sum().item()) <= 4e-3 * c + 1e-6             # sum_v (onehot - p) = 0
        else:
            assert torch.count_nonzero(row).item() == 0                         # masked rows are zero


def test_pythia_full_all_sequences():
    w = syn.WORKLOADS["pythia"]
    inp, o, d = run_full(w, 0)
    ref = H.oracle_seq_values(w, 0, 0, w.B)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp (all 256 sequences)")
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), ref["n_tok"])
    loss, logz, eps = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, w.K)
    H.assert_seq_close(o.log_z.cpu().numpy(), logz, "log_z")
    H.assert_seq_close(o.resid.cpu().numpy(), eps, "resid")
    H.assert_seq_close([o.partial[0].item()], [loss], "loss")
    check_groups(w, 0, inp, o, d, [0, 37], n_rows_sample=32)
    check_properties(w, inp, o, d)


def test_redteam_full_unaligned_rows():
    w = syn.WORKLOADS["redteam"]
    inp, o, d = run_full(w, 1)
    ref = H.oracle_seq_values(w, 1, 0, w.B)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], "seq_logp (all 1024 sequences)")
    loss, logz, eps = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, w.K)
    H.assert_seq_close(o.resid.cpu().numpy(), eps, "resid")
    H.assert_seq_close([o.partial[0].item()], [loss], "loss")
    check_groups(w, 1, inp, o, d, [5, 127], n_rows_sample=32)
    check_properties(w, inp, o, d)


def test_rhomath_full_ragged_sampled_groups():
    w = syn.WORKLOADS["rhomath"]
    inp, o, d = run_full(w, 2)
    check_groups(w, 2, inp, o, d, [0, 17, 31], n_rows_sample=24)
    check_properties(w, inp, o, d)


def test_qwen_shard_bench_configuration():
    w = syn.WORKLOADS["qwen_shard"]  # exactly what bench.py times at N=1
    inp, o, d = run_full(w, 0)
    check_groups(w, 0, inp, o, d, [3], n_rows_sample=16)
    check_properties(w, inp, o, d, n_rows=32)
    # bitwise determinism of a second run over the same buffers
    o2, ws2 = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"], w.beta,
                              w.K, float(w.N))
    assert torch.equal(o2.seq_logp, o.seq_logp) and torch.equal(o2.partial, o.partial)
    d2 = tba.vargrad_bwd(inp["logits"], inp["tokens"], inp["mask"], ws2, o2.resid, 2.0 / w.N)
    assert torch.equal(d2.view(torch.int16), d.view(torch.int16))


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


@pytest.mark.parametrize("name,seed,groups", [("gsm8k_t3", 0, [0, 6]), ("gsm8k_k40", 1, [0, 2]),
                                              ("tldr_t4", 2, [3, 7])])
def test_paper_table_batch_shapes_full(name, seed, groups):
    """The paper's own batch shapes (Tables 3 and 4, the K = 40 ablation) at full size."""
    w = syn.WORKLOADS[name]
    inp, o, d = run_full(w, seed)
    ref = H.oracle_seq_values(w, seed, 0, w.B)
    H.assert_seq_close(o.seq_logp.cpu().numpy(), ref["ell"], f"seq_logp (all {w.N} sequences)")
    np.testing.assert_array_equal(o.n_tokens.cpu().numpy(), ref["n_tok"])
    loss, logz, eps = O.vargrad_tb_loss(ref["ell"], ref["ref_logp"], ref["log_reward"], w.beta, w.K)
    H.assert_seq_close(o.log_z.cpu().numpy(), logz, "log_z")
    H.assert_seq_close(o.resid.cpu().numpy(), eps, "resid")
    H.assert_seq_close([o.partial[0].item()], [loss], "loss")
    check_groups(w, seed, inp, o, d, groups, n_rows_sample=16)
    check_properties(w, inp, o, d)


def test_math_t5_two_groups_ragged_2048():
    """Table 5's MATH shape (K = 16, responses up to 2048 tokens, V = 152064): two whole groups
    (20 GB of logits), one compared with the oracle sequence by sequence."""
    w = syn.WORKLOADS["math_t5_shard"]
    inp, o, d = run_full(w, 3, 0, 2)
    check_groups(w, 3, inp, o, d, [1], n_rows_sample=12)
    check_properties(w, inp, o, d, n_rows=32)
