"""The full-size parity harness is not vacuous (CPU): compare_dlogits_rows accepts the oracle's
own rounded rows and rejects a single element moved by 2 bf16 ulps / past the fp32 bar, and
oracle_seq_values (worker pool + C host generator) equals the in-process oracle."""
import dataclasses

import numpy as np
import pytest
import torch

import tba_synth as syn
from oracle import tba_oracle as O

from . import _harness as H


def _case(dtype):
    w = dataclasses.replace(syn.WORKLOADS["pythia"], B=2, K=2, T=3, V=997, dtype=dtype)
    gi = syn.group_inputs(w, 4, 0, w.B)
    z = H.host_logits(w, 4, 0, w.B)
    r = O.vargrad_head(z, gi["tokens"], gi["mask"], gi["ref_logp"], gi["log_reward"], w.beta, w.K)
    return w, gi, r


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_compare_rows_accepts_oracle_and_rejects_one_bad_element(dtype):
    w, gi, r = _case(dtype)
    N, T, V = w.N, w.T, w.V
    dl = r["dlogits"].reshape(N * T, V)
    if dtype == "bf16":
        d = torch.from_numpy(O.round_bf16(dl)).to(torch.bfloat16)
    else:
        d = torch.from_numpy(dl.astype(np.float32))
    rows = np.flatnonzero(gi["mask"].reshape(-1))
    eps_row = np.repeat(r["eps"], T)
    n, ma, mr = H.compare_dlogits_rows(d, w, 4, rows, 0, gi["tokens"].reshape(-1), eps_row, N, sub=2)
    assert n == len(rows) and mr <= 1.0
    bad = d.clone()
    j = int(np.argmax(np.abs(dl[rows[1]])))
    if dtype == "bf16":
        bad.view(torch.int16)[rows[1], j] += 2                                   # two ulps away
    else:
        bad[rows[1], j] += 3e-6 * max(1.0, abs(2 * r["eps"][rows[1] // T] / N))
    with pytest.raises(AssertionError, match="1 elements outside tolerance"):
        H.compare_dlogits_rows(bad, w, 4, rows, 0, gi["tokens"].reshape(-1), eps_row, N, sub=2)


def test_oracle_seq_values_pool_equals_in_process_oracle():
    w, gi, r = _case("bf16")
    ref = H.oracle_seq_values(w, 4, 0, w.B, chunk_rows=2)
    np.testing.assert_array_equal(ref["ell"], r["ell"])
    np.testing.assert_array_equal(ref["n_tok"], r["n_tok"])
