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
# Full-size oracle runs: input rows are regenerated from the seed by tba_synth's C host twin
# (bit-identical to its NumPy twin) in a persistent pool of spawned worker processes (one per
# host core); every value is computed by oracle/ functions (token_logprob_rows, sequence_sums,
# dlogits_row) — the pool only distributes rows.
_POOL = None
RECORD: list = []   # parity maxima per (test, config, seed, quantity); written by conftest


def n_workers() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def pool():
    global _POOL
    if _POOL is None:
        import multiprocessing as mp
        _POOL = ProcessPoolExecutor(n_workers(), mp_context=mp.get_context("spawn"))
    return _POOL


def record(test: str, config: str, seed: int, quantity: str, n: int, max_abs_err: float, max_err_over_tol: float,
           **extra):
    RECORD.append(dict(test=test, config=config, seed=int(seed), quantity=quantity, n=int(n),
                       max_abs_err=float(max_abs_err), max_err_over_tol=float(max_err_over_tol), **extra))


def _rows_lp(args):
    seed, V, dtype, rows, toks, inv_temp = args
    return O.token_logprob_rows(syn.logits_rows_f64_host(seed, V, rows, dtype), toks, inv_temp)


def oracle_seq_values(w: syn.Workload, seed: int, g0: int, ng: int, chunk_rows: int = 64, inv_temp: float = 1.0):
    """Oracle a1-a2 for groups g0..g0+ng-1 (only valid rows are evaluated). Returns
    dict(ell, n_tok, lse [N, T], tokens, mask, ref_logp, log_reward)."""
    gi = syn.group_inputs(w, seed, g0, ng)
    tok, mask = gi["tokens"], gi["mask"]
    N, T = tok.shape
    base = g0 * w.K * T
    valid = np.flatnonzero(mask.reshape(-1))
    jobs = [(seed, w.V, w.dtype, base + valid[i:i + chunk_rows], tok.reshape(-1)[valid[i:i + chunk_rows]], inv_temp)
            for i in range(0, len(valid), chunk_rows)]
    res = list(pool().map(_rows_lp, jobs)) if len(jobs) > 1 else [_rows_lp(j) for j in jobs]
    lp = np.full(N * T, np.nan)
    lse = np.full(N * T, np.nan)
    pos = 0
    for a, b in res:
        v = valid[pos:pos + len(a)]
        lp[v], lse[v] = a, b
        pos += len(a)
    ell, ntok = O.sequence_sums(lp.reshape(N, T), mask)
    return dict(ell=ell, n_tok=ntok, lse=lse.reshape(N, T), **gi)


def oracle_token_lp(w: syn.Workload, seed: int, g0: int, ng: int, chunk_rows: int = 64):
    """Oracle per-token log-probs lp [N, T] (0 at masked positions) for groups g0..g0+ng-1, computed
    by token_logprob_rows on regenerated rows in the worker pool."""
    gi = syn.group_inputs(w, seed, g0, ng)
    tok, mask = gi["tokens"], gi["mask"]
    N, T = tok.shape
    base = g0 * w.K * T
    valid = np.flatnonzero(mask.reshape(-1))
    jobs = [(seed, w.V, w.dtype, base + valid[i:i + chunk_rows], tok.reshape(-1)[valid[i:i + chunk_rows]], 1.0)
            for i in range(0, len(valid), chunk_rows)]
    res = list(pool().map(_rows_lp, jobs)) if len(jobs) > 1 else [_rows_lp(j) for j in jobs]
    lp = np.zeros(N * T)
    pos = 0
    for a, _ in res:
        lp[valid[pos:pos + len(a)]] = a
        pos += len(a)
    return lp.reshape(N, T), gi


def _cmp_rows(args):
    """Worker: compare GPU dlogits rows (read from a /dev/shm memmap) with oracle dlogits_row."""
    path, shape, gdt, i0, i1, seed, V, in_dt, rows, toks, eps, n_global, grad_out, out_dt, kind, inv_temp = args
    mm = np.memmap(path, dtype=np.uint16 if gdt == "bf16" else np.float32, mode="r", shape=shape)
    g = mm[i0:i1]
    g = syn.bf16_bits_to_f64(g) if gdt == "bf16" else g.astype(np.float64)
    z = syn.logits_rows_f64_host(seed, V, rows, in_dt)
    n_bad, max_abs, max_ratio, worst = 0, 0.0, 0.0, None
    for i in range(len(rows)):
        if kind == "tbap":  # eps holds the per-token coefficient, n_global the token count
            want = O.tbap_dlogits_row(z[i], int(toks[i]), float(eps[i]), n_global, grad_out)
            c = -float(eps[i]) / n_global * grad_out
        else:
            want = O.dlogits_row(z[i], int(toks[i]), float(eps[i]), n_global, grad_out, inv_temp)
            c = inv_temp * 2.0 * float(eps[i]) / n_global * grad_out
        if out_dt == "bf16":
            rb = O.round_bf16(want)
            err = np.abs(g[i] - rb)
            ratio = err / O.bf16_ulp(rb)
            ftz = 2.0 ** -126 * max(1.0, abs(c))   # p flushed below 2^-126 (ex2.approx.ftz), scaled by c
            ratio[(np.abs(g[i]) < ftz) & (np.abs(rb) < ftz)] = 0.0
            ok = ratio <= 1.0
            abs_err = np.abs(g[i] - want)
        else:
            abs_err = np.abs(g[i] - want)
            ratio = abs_err / (2e-6 * max(1.0, abs(c)))
            ok = ratio <= 1.0
        bad = int((~ok).sum())
        if bad and worst is None:
            j = int(np.argmax(ratio))
            worst = (int(rows[i]), j, float(g[i][j]), float(want[j]), c)
        n_bad += bad
        max_abs = max(max_abs, float(abs_err.max()))
        max_ratio = max(max_ratio, float(ratio.max()))
    return n_bad, max_abs, max_ratio, worst


def compare_dlogits_rows(d, w: syn.Workload, seed: int, flat_rows, row_base: int, tokens_flat, eps_of_row,
                         n_global: int, grad_out: float = 1.0, what: str = "", chunk: int = 2048, sub: int = 16,
                         kind: str = "tb", inv_temp: float = 1.0):
    """Element-wise comparison of GPU dlogits rows (``d`` viewed [rows, V], local row indices
    ``flat_rows``, all VALID) with oracle dlogits_row on the regenerated logits (global row =
    row_base + local). tokens_flat / eps_of_row: per local row arrays (kind "tbap": eps_of_row holds
    the per-token TBA' coefficient, n_global the token count, oracle tbap_dlogits_row). Raises on any element
    outside the tolerance; returns (n_rows, max_abs_err, max_err_over_tol)."""
    import torch
    flat_rows = np.asarray(flat_rows, dtype=np.int64)
    V = w.V
    dv = d.reshape(-1, V) if d.is_contiguous() else d.view(-1, V)
    gdt = "bf16" if d.dtype == torch.bfloat16 else "fp32"
    # the GPU rows go to the workers through a memory-mapped file: /dev/shm when it has room (a
    # container's /dev/shm can be 64 MB), else the temp directory; the chunk shrinks to fit
    row_bytes = V * (2 if gdt == "bf16" else 4)
    import tempfile
    d_ = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    free = os.statvfs(d_).f_bavail * os.statvfs(d_).f_frsize
    if free < 4 * row_bytes * min(chunk, max(len(flat_rows), 1)):
        d_ = tempfile.gettempdir()
        free = os.statvfs(d_).f_bavail * os.statvfs(d_).f_frsize
    path = os.path.join(d_, f"tba_parity_{os.getpid()}.bin")
    cap = max(1, min(chunk, len(flat_rows), int(free // (2 * row_bytes))))
    tot_bad, max_abs, max_ratio, worst = 0, 0.0, 0.0, None
    if cap == 0:
        return 0, 0.0, 0.0
    mm = np.memmap(path, dtype=np.uint16 if gdt == "bf16" else np.float32, mode="w+", shape=(cap, V))
    try:
        host = torch.from_numpy(mm.view(np.int16) if gdt == "bf16" else mm)
        for c0 in range(0, len(flat_rows), cap):
            rr = flat_rows[c0:c0 + cap]
            idx = torch.from_numpy(rr).to(d.device)
            rows_dev = dv.index_select(0, idx)
            host[:len(rr)].copy_(rows_dev.view(torch.int16) if gdt == "bf16" else rows_dev)
            mm.flush()
            del rows_dev
            jobs = [(path, (cap, V), gdt, i, min(i + sub, len(rr)), seed, V, w.dtype, row_base + rr[i:i + sub],
                     tokens_flat[rr[i:i + sub]], eps_of_row[rr[i:i + sub]], n_global, grad_out, gdt, kind,
                     inv_temp)
                    for i in range(0, len(rr), sub)]
            for nb, ma, mr, wst in pool().map(_cmp_rows, jobs):
                tot_bad += nb
                max_abs = max(max_abs, ma)
                max_ratio = max(max_ratio, mr)
                worst = worst or wst
    finally:
        del mm
        os.unlink(path)
    if tot_bad:
        raise AssertionError(f"dlogits {what}: {tot_bad} elements outside tolerance; first: global row {worst[0]} "
                             f"col {worst[1]} gpu {worst[2]} oracle {worst[3]} c={worst[4]}")
    return len(flat_rows), max_abs, max_ratio


# --------------------------------------------------------------------------- tolerances
def seq_tols(ell_ref, K, rel=1e-4, abs_=1e-5):
    """Bars for log Z and the residuals, propagated from the per-sequence log-prob bar
    (|d ell_s| <= max(rel |ell_s|, abs_), north_star): log Z_i = mean_j(rho + r/beta - ell_j) and
    eps_s = log Z_i - delta_s are exact fp64 combinations of the ell's, so they inherit
    |d log Z_i| <= mean_j tol(ell_j) and |d eps_s| <= tol(ell_s) + mean_j tol(ell_j)
    (reading R23: log Z of a group can be ~0 while its ell's are ~-2000)."""
    t = np.maximum(rel * np.abs(np.asarray(ell_ref, np.float64)), abs_)
    tz = t.reshape(-1, K).mean(1)
    return tz, t + np.repeat(tz, K)


def assert_close_tol(gpu, ref, tol, what):
    """|gpu - ref| <= tol element-wise (tol an array); returns max err / tol."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = np.maximum(np.asarray(tol, np.float64), np.maximum(1e-4 * np.abs(ref), 1e-5))
    bad = ~((np.abs(gpu - ref) <= tol) | (gpu == ref))
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} mismatches, e.g. idx {i}: gpu {gpu[i]} oracle {ref[i]} tol {tol[i]}")
    return float(np.max(np.abs(gpu - ref) / tol)) if len(ref) else 0.0


def assert_seq_close(gpu, ref, what, rel=1e-4, abs_=1e-5):
    """|gpu - ref| <= max(rel |ref|, abs_) element-wise; returns max err / tol."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = np.maximum(rel * np.abs(ref), abs_)
    bad = ~((np.abs(gpu - ref) <= tol) | (gpu == ref))
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} mismatches, e.g. idx {i}: gpu {gpu[i]} oracle {ref[i]}")
    return float(np.max(np.abs(gpu - ref) / tol)) if len(ref) else 0.0


def assert_dlogits_close(gpu_row, ref_row, c_seq, dtype: str, what=""):
    """bf16: within 1 bf16 ulp of the oracle's bf16 value (or both below max(1,|c|) 2^-126: the kernel's
    ex2.approx.ftz flushes p below 2^-126, and c scales what is left);
    fp32: |diff| <= 2e-6 * max(1, |c_seq|) (reading R9)."""
    g = np.asarray(gpu_row, np.float64)
    r = np.asarray(ref_row, np.float64)
    if dtype == "bf16":
        rb = O.round_bf16(r)
        ftz = 2.0 ** -126 * max(1.0, abs(c_seq))   # p flushed below 2^-126 (ex2.approx.ftz), scaled by c
        ok = (np.abs(g - rb) <= O.bf16_ulp(rb)) | ((np.abs(g) < ftz) & (np.abs(rb) < ftz))
    else:
        ok = np.abs(g - r) <= 2e-6 * max(1.0, abs(c_seq))
    if not ok.all():
        i = np.flatnonzero(~ok)[:5]
        raise AssertionError(f"dlogits {what}: {(~ok).sum()} mismatches at {i}: gpu {g[i]} oracle {r[i]} c={c_seq}")
    return float(np.max(np.abs(g - r))) if len(r) else 0.0
