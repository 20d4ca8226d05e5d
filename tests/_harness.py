"""Parity harness (test infrastructure): builds device inputs from tba_synth, runs the CUDA
path through the package's C-ABI binding, and evaluates the fp64 oracle on the same
(bf16-rounded) inputs regenerated on the host by tba_synth's NumPy twin."""
from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

import tba_synth as syn
from oracle import tba_oracle as O

TORCH_DT = None


def torch_dtype(name):
    import torch
    return {"bf16": torch.bfloat16, "fp32": torch.float32}[name]


def device_inputs(w: syn.Workload, seed: int, g0: int = 0, ng: int | None = None, row_stride: int | None = None,
                  device="cuda"):
    """Inputs for groups g0..g0+ng-1 on the device. logits [N, T, V] view of an
    [N, T, row_stride] buffer whose padding holds NaN."""
    import torch
    ng = w.B if ng is None else ng
    gi = syn.group_inputs(w, seed, g0, ng)
    N, T, V = ng * w.K, w.T, w.V
    rs = row_stride or V
    buf = torch.empty((N, T, rs), dtype=torch_dtype(w.dtype), device=device)
    if N * T:
        syn.fill_logits_cuda(buf.view(N * T, rs)[:, :V], seed, g0 * w.K * T, V)  # padding <- NaN
    return dict(
        logits=buf[:, :, :V],
        tokens=torch.from_numpy(gi["tokens"]).to(device),
        mask=torch.from_numpy(gi["mask"]).to(device),
        ref_logp=torch.from_numpy(gi["ref_logp"]).to(device),
        log_reward=torch.from_numpy(gi["log_reward"]).to(device),
        host=gi,
    )


def host_logits(w: syn.Workload, seed: int, g0: int, ng: int) -> np.ndarray:
    N = ng * w.K
    rows = np.arange(g0 * w.K * w.T, (g0 * w.K + N) * w.T)
    return syn.logits_rows_f64(seed, w.V, rows, w.dtype).reshape(N, w.T, w.V)


# --------------------------------------------------------------------------- parallel oracle
def _rows_lp(args):
    seed, V, dtype, rows, toks = args
    z = syn.logits_rows_f64(seed, V, rows, dtype)
    out = np.empty(len(rows))
    lse = np.empty(len(rows))
    for i in range(len(rows)):
        out[i], lse[i] = O.token_logprob(z[i], int(toks[i]))
    return out, lse


def oracle_seq_values(w: syn.Workload, seed: int, g0: int, ng: int, workers: int | None = None,
                      chunk_rows: int = 64):
    """Oracle a1-a3 for groups g0..g0+ng-1, regenerating rows from the seed in worker
    processes (only valid rows are evaluated). Returns dict(ell, n_tok, log_z, eps,
    lse_by_row)."""
    gi = syn.group_inputs(w, seed, g0, ng)
    tok, mask = gi["tokens"], gi["mask"]
    N, T = tok.shape
    base = g0 * w.K * T
    valid = np.flatnonzero(mask.reshape(-1))
    jobs = []
    for i in range(0, len(valid), chunk_rows):
        v = valid[i:i + chunk_rows]
        jobs.append((seed, w.V, w.dtype, base + v, tok.reshape(-1)[v]))
    workers = workers or max(1, len(os.sched_getaffinity(0)))
    lp = np.zeros(N * T)
    lse = np.full(N * T, np.nan)
    if workers > 1 and len(jobs) > 1:
        with ProcessPoolExecutor(workers) as ex:
            res = list(ex.map(_rows_lp, jobs))
    else:
        res = [_rows_lp(j) for j in jobs]
    pos = 0
    for a, b in res:
        v = valid[pos:pos + len(a)]
        lp[v], lse[v] = a, b
        pos += len(a)
    lp = lp.reshape(N, T)
    ell = np.array([math.fsum(lp[s][mask[s] == 1]) for s in range(N)])
    ntok = mask.sum(1).astype(np.int64)
    return dict(ell=ell, n_tok=ntok, lse=lse.reshape(N, T), **gi)


# --------------------------------------------------------------------------- tolerances
def assert_seq_close(gpu, ref, what, rel=1e-4, abs_=1e-5):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = np.maximum(rel * np.abs(ref), abs_)
    bad = ~((np.abs(gpu - ref) <= tol) | (gpu == ref))
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} mismatches, e.g. idx {i}: gpu {gpu[i]} oracle {ref[i]}")
    return float(np.max(np.abs(gpu - ref) / np.maximum(np.abs(ref), abs_ / rel))) if len(ref) else 0.0


def assert_dlogits_close(gpu_row, ref_row, c_seq, dtype: str, what=""):
    """bf16: within 1 bf16 ulp of the oracle's bf16 value (or both below 2^-126);
    fp32: |diff| <= 2e-6 * max(1, |c_seq|) (reading R9)."""
    g = np.asarray(gpu_row, np.float64)
    r = np.asarray(ref_row, np.float64)
    if dtype == "bf16":
        rb = O.round_bf16(r)
        ok = (np.abs(g - rb) <= O.bf16_ulp(rb)) | ((np.abs(g) < 2.0 ** -126) & (np.abs(rb) < 2.0 ** -126))
    else:
        ok = np.abs(g - r) <= 2e-6 * max(1.0, abs(c_seq))
    if not ok.all():
        i = np.flatnonzero(~ok)[:5]
        raise AssertionError(f"dlogits {what}: {(~ok).sum()} mismatches at {i}: gpu {g[i]} oracle {r[i]} c={c_seq}")
    return float(np.max(np.abs(g - r))) if len(r) else 0.0
