"""fp64 CPU ORACLE for the VarGrad trajectory-balance loss head (TBA, arXiv 2503.18929).

TEST INFRASTRUCTURE ONLY. Nothing on the product path may import, call or execute this
module: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
leg / ``--impl reference`` arm use it. It shares no code with the CUDA path (it imports
only NumPy and the standard library); inputs come from ``tba_synth`` (which holds no
arithmetic of the method) or from the tests themselves.

Citations: ``P:L`` = /root/reference/PAPER.md line L (LaTeX source of the paper),
``S:L`` = SPEC.md line L. Equation numbers are by LaTeX environment count:
Eq. 2 ``eq:opt_policy`` P:99-102, Eq. 4 ``eq:logZ`` P:122-130, Eq. 5 ``eq:vargrad``
P:132-141, Eq. 7 ``eq:tba_update`` P:159-176, Appendix A (gradient) P:420-477.

Notation: sequences s = i*K + j (group-major); rows (s, t); z a logits
row; y the sampled token; mu the response mask; ell_s = log pi_theta(y_s | x);
rho_s = log pi_ref(y_s | x); r_s = r_phi(y_s; x).

What the method computes is its definition (Eqs. 4-5 and their exact gradient); there is
no approximation to reproduce, so this file is that definition written out in fp64, in
the paper's order, with no blocking, fusion or reordering.

Pins (tests/test_oracle.py): worked values of S:52, S:53, S:70, S:133, S:143, S:152;
the closed form log Z = log(0.5e + 0.5) at pi_theta = pi* (Eq. 2); softmax rows sum to 1
within 1e-12; shift invariance; scipy's logsumexp; brute-force products of
probabilities; L = mean within-group population variance; per-group shift invariance;
the independent Appendix-A advantage form; central finite differences of the loss;
token_logprob_rows + sequence_sums against the brute-force product row by row; dlogits_row
against central differences of token_logprob, the S:133 worked rows and ``dlogits``.
TBA' (Eq. 16) pins (tests/test_oracle_tbap.py): Dr. GRPO equality at beta = 0 on-policy
(P:616), the Eq. 7 / Eq. 16 link A = -beta*eps, clip/IcePop worked values, the band
(0, inf) no-op, per-group shift invariance, finite differences with coefficients held fixed.
LM-head pins (tests/test_oracle_lmhead.py): brute-force triple loops on tiny inputs, equal
weight rows (lp = -ln V for any hidden state), one-hot weight rows (closed form), invariance
to adding a common vector to every weight row, temperature = scaling the weight; its
backward (lmhead_grads): central finite differences of the loss in h and W, the zero
vocabulary sum of dW (softmax minus one-hot sums to 0), dH = 0 for equal weight rows.
Every function below is pinned by at least one of them ("parity unpinned": none).
"""
from __future__ import annotations

import math

import numpy as np


# ----------------------------------------------------------------------------- a1
def log_softmax_row(z: np.ndarray) -> tuple[np.ndarray, float]:
    """log softmax of one logits row in fp64, max-subtracted ("numerically stable").

    Returns (log-probabilities [V], lse). The sum over the vocabulary is NumPy's
    pairwise summation in fp64 (sequential fp64 could breach the
    1e-12 row-sum pin at V = 152064). A row with no finite entry has lse = -inf.
    """
    z = np.asarray(z, dtype=np.float64)
    m = np.max(z)
    if not np.isfinite(m):
        if m == -np.inf:
            return np.full(z.shape, np.nan), -np.inf
        return np.full(z.shape, np.nan), np.nan
    lse = m + math.log(np.sum(np.exp(z - m)))
    return z - lse, lse


def token_logprob(z: np.ndarray, y: int) -> tuple[float, float]:
    """log softmax(z)[y] and the row's lse (paper: the per-token factor of
    log pi_theta(y|x) in Eqs. 4-5)."""
    V = len(z)
    if not (0 <= y < V):
        raise ValueError(f"token {y} out of range [0, {V})")  # S:50 invalid-input
    lp, lse = log_softmax_row(z)
    return float(lp[y]), lse


# ----------------------------------------------------------------------------- a2
def token_logprob_rows(z_rows: np.ndarray, tokens, inv_temp: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """``token_logprob`` of each row of z_rows [n, V] at its token (tokens [n]): the per-token
    terms of log pi_theta(y|x) (Eqs. 4-5) for a batch of VALID rows, wherever they come from
    (the full-size harness regenerates sampled rows from the seed). ``inv_temp`` a: the
    temperature-scaled policy log softmax(a z) (NEXT 4). Returns (lp [n], lse [n])."""
    n = len(tokens)
    lp = np.empty(n)
    lse = np.empty(n)
    for i in range(n):
        lp[i], lse[i] = token_logprob(inv_temp * np.asarray(z_rows[i], np.float64), int(tokens[i]))
    return lp, lse


def sequence_sums(lp: np.ndarray, mask: np.ndarray):
    """a2: ell_s = sum_{t: mu=1} lp_{s,t} (``math.fsum``, exact) and n_tok_s = sum_t mu_{s,t}.
    lp [N, T] holds the token log-probs at valid positions (other entries are ignored)."""
    N = lp.shape[0]
    ell = np.array([math.fsum(lp[s][mask[s] == 1]) for s in range(N)])
    ntok = np.asarray(mask).sum(1).astype(np.int64)
    return ell, ntok


def seq_logprob(logits: np.ndarray, tokens: np.ndarray, mask: np.ndarray):
    """ell_s = sum_t mu_{s,t} log softmax(z_{s,t})[y_{s,t}] and n_tok_s = sum_t mu_{s,t}.

    logits [N, T, V] (fp64-convertible), tokens [N, T] int, mask [N, T] 0/1. Tokens at
    masked positions are ignored (reading R5). ``token_logprob_rows`` over the
    valid rows, then ``sequence_sums``. Returns (ell [N] fp64, n_tok [N] int64,
    lse [N, T] fp64 with NaN at masked positions)."""
    N, T = tokens.shape
    lp = np.zeros((N, T))
    lse = np.full((N, T), np.nan)
    valid = np.asarray(mask).reshape(-1) == 1
    if valid.any():
        z = np.asarray(logits).reshape(N * T, -1)[valid]
        lpv, lsev = token_logprob_rows(z, np.asarray(tokens).reshape(-1)[valid])
        lp.reshape(-1)[valid] = lpv
        lse.reshape(-1)[valid] = lsev
    ell, ntok = sequence_sums(lp, mask)
    return ell, ntok, lse


# ----------------------------------------------------------------------------- a3
def _check_config(N: int, beta: float, K: int):
    if not (math.isfinite(beta) and beta > 0):
        raise ValueError("invalid-config: beta must be finite and > 0 (S:131)")
    if K < 2:
        raise ValueError("invalid-config: K must be >= 2 (S:140)")
    if N % K:
        raise ValueError("invalid-arg: N must be a multiple of K")


def log_z_hat(ell, ref_logp, log_reward, beta: float, K: int) -> np.ndarray:
    """Eq. 4: log Z(x_i) = (1/K) sum_j (log pi_ref - log pi_theta + r/beta).

    Inputs are per-sequence in group-major order (s = i*K + j). Returns [B] fp64."""
    ell = np.asarray(ell, np.float64)
    _check_config(len(ell), beta, K)
    delta = np.asarray(ref_logp, np.float64) - ell + np.asarray(log_reward, np.float64) / beta
    B = len(ell) // K
    return np.array([math.fsum(delta[i * K:(i + 1) * K]) / K for i in range(B)])


def vargrad_tb_loss(ell, ref_logp, log_reward, beta: float, K: int, n_global: int | None = None):
    """Eq. 5: L = 1/(BK) sum_ij (SG[log Z_i] + log pi_theta - log pi_ref - r/beta)^2.

    Returns (L, log_z [B], eps [N]) with eps_s = log Z_i + ell_s - rho_s - r_s/beta, the
    residual inside the square. ``n_global`` replaces BK when this batch is one shard
    of a larger one (reading R2); default BK = len(ell)."""
    ell = np.asarray(ell, np.float64)
    N = len(ell)
    logz = log_z_hat(ell, ref_logp, log_reward, beta, K)
    eps = np.empty(N)
    for s in range(N):
        i = s // K
        eps[s] = logz[i] + ell[s] - float(ref_logp[s]) - float(log_reward[s]) / beta
    n = N if n_global is None else n_global
    loss = math.fsum(eps * eps) / n
    return loss, logz, eps


def advantages(ell, ref_logp, log_reward, beta: float, K: int) -> np.ndarray:
    """Appendix A: A_ij = (r_ij - rbar_i) - beta (KL_ij - KLbar_i), with
    KL_ij = log pi_theta - log pi_ref. Independent of ``vargrad_tb_loss``; used to pin the
    residual through the identity A = -beta * eps."""
    ell = np.asarray(ell, np.float64)
    _check_config(len(ell), beta, K)
    r = np.asarray(log_reward, np.float64)
    kl = ell - np.asarray(ref_logp, np.float64)
    A = np.empty_like(ell)
    for i in range(len(ell) // K):
        sl = slice(i * K, (i + 1) * K)
        A[sl] = (r[sl] - r[sl].mean()) - beta * (kl[sl] - kl[sl].mean())
    return A


# ----------------------------------------------------------------------------- a5
def grad_logprob_row(z: np.ndarray, y: int) -> np.ndarray:
    """d log softmax(z)[y] / dz = onehot(y) - softmax(z).

    The token's entry 1 - p_y is formed as sum_{v != y} p_v (the same quantity: the softmax sums
    to 1), so it keeps its relative accuracy when p_y -> 1 instead of cancelling in fp64."""
    lp, _ = log_softmax_row(z)
    p = np.exp(lp)
    g = -p
    g[y] = np.sum(np.delete(p, y))
    return g


def dlogits(logits, tokens, mask, eps, n_global: int, grad_out: float = 1.0) -> np.ndarray:
    """dL/dz for Eq. 5 (Appendix A: grad L = (1/BK) sum -2(...) grad log pi, the
    bracket being -eps):  dz_{s,t,v} = mu_{s,t} * (2 eps_s / N) * grad_out * (1[v = y] - p_v).

    Masked rows are exactly 0. Returns fp64 [N, T, V]."""
    N, T = tokens.shape
    V = logits.shape[-1]
    out = np.zeros((N, T, V), dtype=np.float64)
    for s in range(N):
        g = 2.0 * float(eps[s]) / n_global * grad_out
        for t in range(T):
            if mask[s, t]:
                out[s, t] = g * grad_logprob_row(logits[s, t], int(tokens[s, t]))
    return out


def dlogits_row(z, y: int, eps_s: float, n_global: int, grad_out: float = 1.0, inv_temp: float = 1.0) -> np.ndarray:
    """One valid row of ``dlogits`` (for sampled-row comparison at full size); with ``inv_temp`` a
    the chain rule through log softmax(a z): a (2 eps / N) g (onehot - softmax(a z))."""
    return inv_temp * (2.0 * eps_s / n_global * grad_out) * grad_logprob_row(inv_temp * np.asarray(z, np.float64), y)


# ----------------------------------------------------------------------------- full head
def vargrad_head(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int,
                 n_global: int | None = None, grad_out: float = 1.0, want_grad: bool = True,
                 inv_temp: float = 1.0, log_z=None):
    """Steps a1-a5 of SURVEY §8(a) on one (shard of a) batch. Returns a dict with
    ell, n_tok, log_z, eps, loss (normalised by n_global), partial = [sum eps^2 / n_global,
    N, B], and dlogits (fp64) if requested.

    Variants: ``inv_temp`` a: log pi = log softmax(a z), so the chain
    rule gives dz = a (2 eps/N) g (onehot - softmax(a z)); ``log_z`` (length B): a learned
    log Z(x_i) (Eq. 3) replaces the Eq. 4 estimate, and d_log_z = sum_j 2 eps/N g."""
    scaled = np.asarray(logits, np.float64) * inv_temp
    ell, ntok, lse = seq_logprob(scaled, tokens, mask)
    N = len(ell)
    n = N if n_global is None else n_global
    if log_z is None:
        loss, logz, eps = vargrad_tb_loss(ell, ref_logp, log_reward, beta, K, n)
    else:
        loss, logz, eps = tb_learned_z_loss(ell, ref_logp, log_reward, beta, K, log_z, n)
    out = dict(ell=ell, n_tok=ntok, lse=lse, log_z=logz, eps=eps, loss=loss,
               partial=np.array([loss, float(N), float(N // K)]))
    if log_z is not None:
        out["d_log_z"] = learned_log_z_grad(eps, K, n, grad_out)
    if want_grad:
        out["dlogits"] = inv_temp * dlogits(scaled, tokens, mask, eps, n, grad_out)
    return out


def learned_log_z_grad(eps, K: int, n_global: int, grad_out: float = 1.0) -> np.ndarray:
    """dL/dlog Z(x_i) for a learned log Z (Eq. 3, no stop-gradient): (2 / N) g sum_j eps_{iK+j}."""
    N = len(eps)
    return np.array([2.0 * math.fsum(eps[i * K:(i + 1) * K]) / n_global * grad_out for i in range(N // K)])


def tb_learned_z_loss(ell, ref_logp, log_reward, beta: float, K: int, log_z, n_global: int | None = None):
    """Eq. 3 with R(y;x) = pi_ref(y|x) exp(r/beta), averaged over the batch
    like Eq. 5: L = 1/(BK) sum_ij (log Z(x_i) + log pi_theta - log pi_ref - r/beta)^2 with a
    learned log Z(x_i) (no stop-gradient). Returns (L, log_z, eps)."""
    ell = np.asarray(ell, np.float64)
    _check_config(len(ell), beta, K)
    N = len(ell)
    lz = np.asarray(log_z, np.float64)
    eps = np.array([lz[s // K] + ell[s] - float(ref_logp[s]) - float(log_reward[s]) / beta for s in range(N)])
    n = N if n_global is None else n_global
    return math.fsum(eps * eps) / n, lz.copy(), eps


# ----------------------------------------------------------------------------- TBA' (NEXT 1)
def is_weight(lam: float, mode: str, lo: float, hi: float) -> float:
    """IS weight of Eq. 16: 'none' -> 1; 'clip' -> min(max(lam, lo), hi) (CISPO bounds 0/8,
    Table 5; the display's min(lambda, 8)); 'icepop' -> lam inside [lo, hi] else 0
    (masking the gradient of tokens with large or small ratios; R14)."""
    if mode == "none":
        return 1.0
    if mode == "clip":
        return min(max(lam, lo), hi)
    if mode == "icepop":
        return lam if lo <= lam <= hi else 0.0
    raise ValueError(mode)


def tbap_coefficients(lp, mask, gen_logp, ref_logp, log_reward, beta: float, K: int, is_mode: str = "clip",
                      is_lo: float = 0.0, is_hi: float = 8.0, n_tok_global: int | None = None):
    """Eq. 16 from the per-token log-probs lp [N, T] (valid positions only are read),
    step by step in the paper's notation:
      lambda_t = pi_theta(y_t)/pi_gen(y_t) = exp(lp_t - gen_t)      per token
      log Lambda_j = ell_j - rho_j,  ell_j = sum_t lp_t              (sequence_sums)
      A_j = (r_j - rbar) - beta (log Lambda_j - mean_j log Lambda)  per group of K
      coef_t = w(lambda_t) A_j                                       (a stop-gradient constant)
    and the surrogate loss L' = -(1/n_tok) sum_t coef_t lp_t (GRPO-style normalisation, P:708;
    DESIGN.md R15). Returns dict(ell, n_tok, adv, coef [N, T], loss, partial)."""
    if not (math.isfinite(beta) and beta >= 0):
        raise ValueError("invalid-config: beta must be finite and >= 0")
    N, T = np.shape(mask)
    if K < 2:
        raise ValueError("invalid-config: K must be >= 2")
    if N % K:
        raise ValueError("invalid-arg: N must be a multiple of K")
    ell, ntok = sequence_sums(lp, mask)
    ref = np.asarray(ref_logp, np.float64)
    r = np.asarray(log_reward, np.float64)
    A = np.empty(N)
    for i in range(N // K):
        sl = slice(i * K, (i + 1) * K)
        logL = ell[sl] - ref[sl]
        A[sl] = (r[sl] - r[sl].mean()) - beta * (logL - logL.mean())
    coef = np.zeros((N, T))
    for s in range(N):
        for t in range(T):
            if mask[s, t]:
                lam = math.exp(lp[s, t] - float(gen_logp[s, t]))
                coef[s, t] = is_weight(lam, is_mode, is_lo, is_hi) * A[s]
    n = int(ntok.sum()) if n_tok_global is None else n_tok_global
    terms = [coef[s, t] * lp[s, t] for s in range(N) for t in range(T) if mask[s, t]]
    loss = -math.fsum(terms) / n
    return dict(ell=ell, n_tok=ntok, adv=A, coef=coef, loss=loss,
                partial=np.array([loss, float(ntok.sum()), float(N)]))


def tbap_dlogits_row(z, y: int, coef_t: float, n_tok: int, grad_out: float = 1.0) -> np.ndarray:
    """One valid row of the TBA' surrogate's gradient: -(coef_t / n_tok) g (onehot(y) - softmax(z))."""
    return -(coef_t / n_tok) * grad_out * grad_logprob_row(z, y)


def tbap_head(logits, tokens, mask, gen_logp, ref_logp, log_reward, beta: float, K: int, is_mode: str = "clip",
              is_lo: float = 0.0, is_hi: float = 8.0, n_tok_global: int | None = None, grad_out: float = 1.0,
              want_grad: bool = True):
    """TBA' token-level rule, Eq. 16: grad J = sum_j sum_t sg(w(lambda_t) A_j)
    grad log pi_theta(y_t), normalised by the number of valid tokens (GRPO-style; R15).
    token_logprob_rows over the valid rows, then tbap_coefficients; dlogits (if requested) =
    tbap_dlogits_row per valid row. Returns the surrogate loss L' = -(1/n_tok) sum coef_t lp_t
    (whose gradient is -grad J / n_tok), lp, ell, n_tok, A, coef [N, T] and dlogits."""
    N, T = tokens.shape
    lp = np.zeros((N, T))
    valid = np.asarray(mask).reshape(-1) == 1
    if valid.any():
        lp.reshape(-1)[valid] = token_logprob_rows(np.asarray(logits).reshape(N * T, -1)[valid],
                                                   np.asarray(tokens).reshape(-1)[valid])[0]
    out = tbap_coefficients(lp, mask, gen_logp, ref_logp, log_reward, beta, K, is_mode, is_lo, is_hi, n_tok_global)
    out["lp"] = lp
    n = int(out["n_tok"].sum()) if n_tok_global is None else n_tok_global
    if want_grad:
        d = np.zeros(np.shape(logits))
        for s in range(N):
            for t in range(T):
                if mask[s, t]:
                    d[s, t] = tbap_dlogits_row(logits[s, t], int(tokens[s, t]), out["coef"][s, t], n, grad_out)
        out["dlogits"] = d
    return out


# ----------------------------------------------------------------------------- bf16
def round_bf16(x) -> np.ndarray:
    """Round fp64 values to the nearest bf16 value (ties to even), returned as fp64.

    bf16 has 8 significant bits and fp32's exponent range; below 2^-126 the spacing is
    fixed at 2^-133 (subnormals). Overflow is not handled (|x| < 3e38 assumed)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    nz = (x != 0) & np.isfinite(x)
    _, e = np.frexp(x[nz])                 # x = f * 2^e, 0.5 <= |f| < 1
    e = np.maximum(e, -125)                # subnormal range: fixed ulp 2^-133
    ulp = np.ldexp(1.0, e - 8)
    out[nz] = np.rint(x[nz] / ulp) * ulp   # rint = round half to even; /ulp is exact
    out[~np.isfinite(x)] = x[~np.isfinite(x)]
    return out


def bf16_ulp(x) -> np.ndarray:
    """Spacing of bf16 values at |x| (for the 1-ulp dlogits tolerance)."""
    x = np.abs(np.asarray(x, dtype=np.float64))
    _, e = np.frexp(np.where(x > 0, x, 1.0))
    e = np.where(x > 0, np.maximum(e, -125), -125)
    return np.ldexp(1.0, e - 8)


# ----------------------------------------------------------------------------- NEXT 3: from hidden states
def lmhead_logits(hidden: np.ndarray, weight: np.ndarray) -> np.ndarray:
    """z_{r,v} = sum_i h_{r,i} W_{v,i}: the LM-head contraction that ends the "single forward
    pass" of P:202 (the logits every a1 step consumes), in fp64 (a library matmul of the
    exact fp64 values of the bf16 inputs). hidden [R, d], weight [V, d] -> [R, V]."""
    return np.asarray(hidden, np.float64) @ np.asarray(weight, np.float64).T


def lmhead_token_logprob(hidden: np.ndarray, weight: np.ndarray, tokens, inv_temp: float = 1.0,
                         chunk: int = 8192) -> np.ndarray:
    """log softmax(inv_temp * W h_r)[y_r] for every row r of hidden [R, d] (tokens [R]), fp64.
    The weight may be a callable ``weight(v0, v1) -> [v1 - v0, d]`` (rows generated on demand,
    for vocabularies too large to hold in fp64); the logits are then built chunk by chunk
    (the chunking only splits the matmul's output columns; every z is the same dot product)."""
    hidden = np.asarray(hidden, np.float64)
    if callable(weight):
        V = weight.vocab
        parts = []
        for v0 in range(0, V, chunk):
            parts.append(lmhead_logits(hidden, weight(v0, min(V, v0 + chunk))))
        z = np.concatenate(parts, axis=1)
    else:
        z = lmhead_logits(hidden, weight)
    out = np.empty(len(hidden))
    for r in range(len(hidden)):
        out[r] = token_logprob(inv_temp * z[r], int(tokens[r]))[0]
    return out


def lmhead_seq_logprob(hidden: np.ndarray, weight: np.ndarray, tokens: np.ndarray, mask: np.ndarray,
                       inv_temp: float = 1.0):
    """seq_logprob of the logits z = inv_temp * W h (hidden [N, T, d]); returns (ell, n_tok)."""
    N, T, d = np.shape(hidden)
    z = inv_temp * lmhead_logits(np.reshape(hidden, (N * T, d)), weight).reshape(N, T, -1)
    ell, ntok, _ = seq_logprob(z, tokens, mask)
    return ell, ntok


def lmhead_grads(hidden: np.ndarray, weight: np.ndarray, dz: np.ndarray):
    """Backward through z = W h (NEXT 3): the chain rule applied to App. A's dL/dz:
        dL/dh_r = sum_v dz_{r,v} W_v   and   dL/dW_v = sum_r dz_{r,v} h_r,
    i.e. dH = dZ W and dW = dZ^T H (library matmuls in fp64). hidden [R, d], weight [V, d],
    dz [R, V] (e.g. ``vargrad_head(...)["dlogits"]`` reshaped) -> (dH [R, d], dW [V, d])."""
    H = np.asarray(hidden, np.float64)
    W = np.asarray(weight, np.float64)
    Z = np.asarray(dz, np.float64)
    return Z @ W, Z.T @ H
