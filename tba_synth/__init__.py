"""Seeded synthetic inputs for the VarGrad TB-loss head — shared by the oracle and the CUDA path.

This module is the ONLY code both sides use. It holds no arithmetic of the method
(no softmax, no log-probabilities, no loss): just an integer counter-based hash,
the recipe that turns hash bits into logits/tokens/masks/rewards, and the workload
presets. Its CUDA twin (``tba_synth/csrc/synth.cu`` -> ``libtba_synth.so``) produces
bit-identical logits on the device for the sizes the host cannot hold.

Recipe (DESIGN.md §"Input recipe"):

* hash: SplitMix64 finaliser, counter-based. ``key(seed, stream)`` selects an
  independent stream; element ``i`` of a stream is ``mix64(key + (i+1)*GAMMA)``,
  i.e. the i-th output of a SplitMix64 generator started at ``key``.
* logits: ``z = (u0+u1+u2+u3 - 131070) * 2^-14`` with ``u_k`` the four 16-bit
  fields of one hash (Irwin–Hall, ~N(0, 2.31^2), |z| <= 8, exact in fp32); the row's
  sampled token gets a peak ``z[y] += b``, ``b in {0,4,8,12}`` (fp32 add, exact);
  bf16 by integer round-to-nearest-even of the fp32 bits. Index = row*V + v, so the
  content does not depend on the row stride; padding columns hold NaN (0x7FC0 /
  0x7FC00000) to prove they are never read.
* tokens: ``y = mulhi(h, V)``; masked positions carry -1 (any value is legal there).
* masks: prefix masks of length ``L_s`` (full T, or uniform on [lo, hi]).
* ref_logp: ``e_V * L_s + U(-20, 20)`` with ``e_V = 6 - (ln V + 2.65)``; log_reward per
  task (binary correctness / reward-model score / sparse red-team log-reward / U(0,1)).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MUL1 = 0xBF58476D1CE4E5B9
MUL2 = 0x94D049BB133111EB
STREAM_MUL = 0xD1B54A32D192ED03

# stream ids (must match tba_synth/csrc/synth.cu)
S_LOGITS, S_TOKENS, S_PEAK, S_LEN, S_REF, S_REWARD, S_BERN = 1, 2, 3, 4, 5, 6, 7

BF16_NAN = 0x7FC0
F32_NAN_BITS = 0x7FC00000


# ----------------------------------------------------------------------------- hash
def mix64_scalar(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * MUL1) & M64
    z = ((z ^ (z >> 27)) * MUL2) & M64
    return z ^ (z >> 31)


def splitmix64_scalar(state: int, i: int) -> int:
    """i-th (0-based) output of SplitMix64 started at ``state`` (pure-Python ints)."""
    return mix64_scalar((state + (i + 1) * GAMMA) & M64)


def stream_key(seed: int, stream: int) -> int:
    return mix64_scalar(mix64_scalar((seed + GAMMA) & M64) ^ ((stream * STREAM_MUL) & M64))


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= np.uint64(MUL1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(MUL2)
    z ^= z >> np.uint64(31)
    return z


def hash64(seed: int, stream: int, idx) -> np.ndarray:
    """Vectorised counter hash: element ``idx`` of stream ``stream`` under ``seed``."""
    key = np.uint64(stream_key(seed, stream))
    i = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64(key + (i + np.uint64(1)) * np.uint64(GAMMA))


def mulhi_u64(h: np.ndarray, n: int) -> np.ndarray:
    """floor(h * n / 2^64) for uint64 h and 0 < n < 2^32, exact."""
    assert 0 < n < (1 << 32)
    h = np.asarray(h, dtype=np.uint64)
    hi = h >> np.uint64(32)
    lo = h & np.uint64(0xFFFFFFFF)
    nn = np.uint64(n)
    return (hi * nn + ((lo * nn) >> np.uint64(32))) >> np.uint64(32)


def unit24(h: np.ndarray) -> np.ndarray:
    """Top 24 bits of the hash as a float64 in [0, 1) (exact in fp32 as well)."""
    return (np.asarray(h, dtype=np.uint64) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


# ----------------------------------------------------------------------------- bf16
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, by integer arithmetic on the bit pattern
    (finite inputs only)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


# ----------------------------------------------------------------------------- presets
@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    B: int               # prompt groups
    K: int               # samples per prompt
    T: int               # padded response length
    V: int               # vocabulary
    dtype: str           # "bf16" | "fp32" logits (and dlogits)
    beta: float
    len_lo: int          # response length L_s ~ U{len_lo..len_hi} (== T for full masks)
    len_hi: int
    reward: str          # "binary" | "rm" | "redteam" | "unit"
    note: str = ""
    d: int = 0           # hidden size of the model's LM head (LM-head-fused path, NEXT 3)

    @property
    def N(self) -> int:
        return self.B * self.K

    def with_groups(self, B: int) -> "Workload":
        return dataclasses.replace(self, B=B)


# BASELINE.json configs; paper anchors in DESIGN.md (§ Input recipe)
WORKLOADS = {
    "toy": Workload("toy", 2, 4, 16, 1000, "fp32", 1.0, 16, 16, "unit",
                    "toy VarGrad TB: 2x4, T=16, V=1000, beta=1, fp32 logits"),
    "pythia": Workload("pythia", 64, 4, 53, 50304, "bf16", 0.05, 53, 53, "rm",
                       "Pythia-410M TL;DR: V=50304, 53-token responses, 64x4"),
    "rhomath": Workload("rhomath", 32, 20, 512, 32000, "bf16", 0.012, 64, 512, "binary",
                        "RhoMath-1B GSM8K: V=32000, <=512-token responses, 32x20"),
    "redteam": Workload("redteam", 128, 8, 20, 50257, "bf16", 0.05, 20, 20, "redteam",
                        "GPT-2 red-teaming: V=50257, 20 tokens, 128x8, sparse log-rewards"),
    "qwen": Workload("qwen", 64, 8, 1024, 152064, "bf16", 0.005, 1024, 1024, "binary",
                     "Qwen2.5-7B MATH: V=152064, 1024 tokens, 64x8 (sharded by group over 8 GPUs)"),
}
# Hidden sizes of the models named in BASELINE.json (their LM heads: d x V, no bias): Qwen2.5-7B
# 3584, Pythia-410M 1024, RhoMath-1B (TinyLlama-1.1B architecture) 2048, GPT-2 small 768.
for _n, _d in (("toy", 64), ("pythia", 1024), ("rhomath", 2048), ("redteam", 768), ("qwen", 3584)):
    WORKLOADS[_n] = dataclasses.replace(WORKLOADS[_n], d=_d)
# The per-GPU shard of the Qwen batch at 8xB200 (8 of the 64 groups).
WORKLOADS["qwen_shard"] = dataclasses.replace(WORKLOADS["qwen"], name="qwen_shard", B=8,
                                              note="Qwen2.5-7B MATH per-GPU shard: 8 groups x K=8, T=1024, V=152064")
# Pythia TL;DR in fp32 logits/dlogits: the paper's PFT runs were fp32 without DeepSpeed.
WORKLOADS["pythia_fp32"] = dataclasses.replace(WORKLOADS["pythia"], name="pythia_fp32", dtype="fp32",
                                               note="Pythia-410M TL;DR shape with fp32 logits (PFT precision, P:593)")
# The paper's own batch shapes (its hyperparameter tables; BASELINE.json's configs differ):
# GSM8K Table 3: 7 prompts x K=20, responses up to 512 tokens, Rho-1B vocabulary.
WORKLOADS["gsm8k_t3"] = dataclasses.replace(WORKLOADS["rhomath"], name="gsm8k_t3", B=7,
                                            note="paper Table 3 (GSM8K): 7 x K=20, T=512, V=32000")
# GSM8K K ablation (`tab:k_ablate`): K=40 with fewer prompts; 140/40 is not whole, so 3 x 40
# (the largest whole-group batch not above Table 3's 140; DESIGN.md R-presets).
WORKLOADS["gsm8k_k40"] = dataclasses.replace(WORKLOADS["rhomath"], name="gsm8k_k40", B=3, K=40,
                                             note="paper K ablation tab:k_ablate (GSM8K): 3 x K=40, T=512, V=32000")
# TL;DR Table 4: 8 prompts x K=20, 128-token responses, Pythia vocabulary.
WORKLOADS["tldr_t4"] = dataclasses.replace(WORKLOADS["pythia"], name="tldr_t4", B=8, K=20, T=128,
                                           len_lo=128, len_hi=128,
                                           note="paper Table 4 (TL;DR): 8 x K=20, T=128, V=50304")
# MATH Table 5: 32 prompts x K=16; responses up to 3072 - 1024 = 2048 tokens, length
# mix unstated: L_s ~ U{256..2048} (DESIGN.md R-presets). The whole batch is 319 GB of bf16
# logits; `math_t5_shard` is its per-GPU share at 8xB200 (4 groups, 39.9 GB).
WORKLOADS["math_t5"] = dataclasses.replace(WORKLOADS["qwen"], name="math_t5", B=32, K=16, T=2048,
                                           len_lo=256, len_hi=2048,
                                           note="paper Table 5 (MATH): 32 x K=16, T<=2048, V=152064")
WORKLOADS["math_t5_shard"] = dataclasses.replace(WORKLOADS["math_t5"], name="math_t5_shard", B=4,
                                                 note="paper Table 5 (MATH) per-GPU shard at 8xB200: "
                                                      "4 x K=16, T<=2048, V=152064")
# One Qwen group (8 x 1024 rows, 2.5 GB of logits): the slice `ncu --set full` replays.
WORKLOADS["qwen_group"] = dataclasses.replace(WORKLOADS["qwen"], name="qwen_group", B=1,
                                              note="one Qwen2.5-7B MATH group: 1 x K=8, T=1024, V=152064 (profiling)")


# ----------------------------------------------------------------------------- generators
def seq_lengths(w: Workload, seed: int, seq0: int = 0, n: int | None = None) -> np.ndarray:
    """Response lengths L_s for global sequences seq0 .. seq0+n-1."""
    n = w.N if n is None else n
    s = np.arange(seq0, seq0 + n, dtype=np.uint64)
    if w.len_lo == w.len_hi:
        return np.full(n, w.len_hi, dtype=np.int64)
    span = w.len_hi - w.len_lo + 1
    return (w.len_lo + mulhi_u64(hash64(seed, S_LEN, s), span)).astype(np.int64)


def raw_tokens(seed: int, V: int, rows) -> np.ndarray:
    """The sampled token of each global row (also where the logit peak sits)."""
    return mulhi_u64(hash64(seed, S_TOKENS, rows), V).astype(np.int64)


def peak_of(seed: int, rows) -> np.ndarray:
    return (4 * (hash64(seed, S_PEAK, rows) & np.uint64(3))).astype(np.float32)


def tokens_and_mask(w: Workload, seed: int, seq0: int = 0, n: int | None = None):
    """tokens int64 [n, T] (-1 where masked) and mask uint8 [n, T] (prefix masks)."""
    n = w.N if n is None else n
    L = seq_lengths(w, seed, seq0, n)
    t = np.arange(w.T, dtype=np.int64)
    mask = (t[None, :] < L[:, None]).astype(np.uint8)
    rows = (np.arange(seq0, seq0 + n, dtype=np.int64)[:, None] * w.T + t[None, :]).astype(np.uint64)
    tok = raw_tokens(seed, w.V, rows)
    tok = np.where(mask == 1, tok, -1).astype(np.int64)
    return tok, mask


def logits_rows_f32(seed: int, V: int, rows) -> np.ndarray:
    """fp32 logits (before any bf16 rounding) for the given global rows: [len(rows), V]."""
    rows = np.asarray(rows, dtype=np.uint64).reshape(-1)
    idx = rows[:, None] * np.uint64(V) + np.arange(V, dtype=np.uint64)[None, :]
    h = hash64(seed, S_LOGITS, idx)
    acc = np.zeros(h.shape, dtype=np.int64)
    for k in range(4):
        acc += ((h >> np.uint64(16 * k)) & np.uint64(0xFFFF)).astype(np.int64)
    z = ((acc - 131070).astype(np.float64) * (2.0 ** -14)).astype(np.float32)
    y = raw_tokens(seed, V, rows)
    b = peak_of(seed, rows)
    r = np.arange(len(rows))
    z[r, y] = (z[r, y] + b).astype(np.float32)
    return z


def logits_rows(seed: int, V: int, rows, dtype: str) -> np.ndarray:
    """Logits rows exactly as stored on the device: uint16 bf16 bits or fp32."""
    z = logits_rows_f32(seed, V, rows)
    if dtype == "bf16":
        return f32_to_bf16_bits(z)
    return z


def logits_rows_f64(seed: int, V: int, rows, dtype: str) -> np.ndarray:
    """The stored logits converted exactly to fp64 (what the oracle consumes)."""
    z = logits_rows(seed, V, rows, dtype)
    if dtype == "bf16":
        return bf16_bits_to_f64(z)
    return z.astype(np.float64)


def ref_logp(w: Workload, seed: int, seq0: int = 0, n: int | None = None) -> np.ndarray:
    """Per-sequence reference log-prob: e_V * L_s + U(-20, 20), fp32-representable."""
    n = w.N if n is None else n
    L = seq_lengths(w, seed, seq0, n)
    e_v = 6.0 - (math.log(w.V) + 2.65)
    u = unit24(hash64(seed, S_REF, np.arange(seq0, seq0 + n, dtype=np.uint64)))
    return (e_v * L + (-20.0 + 40.0 * u)).astype(np.float32).astype(np.float64)


def log_reward(w: Workload, seed: int, seq0: int = 0, n: int | None = None) -> np.ndarray:
    """Per-sequence r_phi (the log of the tilt exp(r_phi), paper Eq. 2), fp32-representable."""
    n = w.N if n is None else n
    s = np.arange(seq0, seq0 + n, dtype=np.uint64)
    u = unit24(hash64(seed, S_REWARD, s))
    if w.reward == "binary":          # correctness reward r in {0, 1}
        r = (hash64(seed, S_BERN, s) >> np.uint64(63)).astype(np.float64)
    elif w.reward == "rm":            # reward-model score
        r = -4.0 + 8.0 * u
    elif w.reward == "redteam":       # sparse log-rewards: 90% U(-12,-4), 10% U(-0.7,0)
        sel = mulhi_u64(hash64(seed, S_BERN, s), 10) == 0
        r = np.where(sel, -0.7 + 0.7 * u, -12.0 + 8.0 * u)
    elif w.reward == "unit":
        r = u
    else:
        raise ValueError(w.reward)
    return r.astype(np.float32).astype(np.float64)


def group_inputs(w: Workload, seed: int, g0: int, ng: int):
    """Everything except logits for groups g0..g0+ng-1 (global group indices)."""
    s0, n = g0 * w.K, ng * w.K
    tok, mask = tokens_and_mask(w, seed, s0, n)
    return dict(tokens=tok, mask=mask, ref_logp=ref_logp(w, seed, s0, n),
                log_reward=log_reward(w, seed, s0, n))


# ----------------------------------------------------------------------------- CUDA twin
_synth_lib = None


def _load_cuda_twin():
    global _synth_lib
    if _synth_lib is None:
        import ctypes
        import os
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtba_synth.so")
        if not os.path.exists(p):
            raise ImportError(f"{p} not built (run __graft_entry__.build())")
        L = ctypes.CDLL(p)
        L.tba_synth_logits.restype = ctypes.c_int
        L.tba_synth_logits.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_void_p]
        L.tba_synth_logits_host.restype = ctypes.c_int
        L.tba_synth_logits_host.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]
        L.tba_synth_bf16.restype = ctypes.c_int
        L.tba_synth_bf16.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        _synth_lib = L
    return _synth_lib


def fill_logits_cuda(out, seed: int, row0: int, V: int, stream: int | None = None):
    """Fill a CUDA tensor ``out`` viewed as [nrows, row_stride] (bf16 or fp32; last dim
    unit-stride, rows uniformly strided) with the logits of global rows row0.. on the
    device. Bit-identical to ``logits_rows`` (columns >= V get NaN)."""
    import torch
    dt = {torch.bfloat16: 0, torch.float32: 1}[out.dtype]
    if out.dim() == 3:
        nrows = out.shape[0] * out.shape[1]
        rs = out.stride(1) if out.shape[1] > 1 else out.stride(0)
    else:
        nrows, rs = out.shape[0], out.stride(0)
    if out.shape[-1] != V or out.stride(-1) != 1:
        raise ValueError("out must be [.., V] with unit stride")
    # fill the padding too: the storage view covers [nrows, rs]
    s = torch.cuda.current_stream(out.device).cuda_stream if stream is None else stream
    rc = _load_cuda_twin().tba_synth_logits(out.data_ptr(), dt, stream_key(seed, S_LOGITS),
                                            stream_key(seed, S_TOKENS), stream_key(seed, S_PEAK), row0, nrows, V,
                                            rs, s)
    if rc:
        raise RuntimeError(f"tba_synth_logits failed ({rc})")
    return out


def logits_rows_host(seed: int, V: int, rows, dtype: str) -> np.ndarray:
    """``logits_rows`` computed by the C host twin (libtba_synth.so, no GPU needed): the same
    element function as the CUDA twin, ~100x faster than the NumPy twin, which pins it bit for
    bit (tests/test_synth.py). For the harness's full-size oracle runs."""
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1))
    out = np.empty((len(rows), V), dtype=np.uint16 if dtype == "bf16" else np.float32)
    if len(rows):
        rc = _load_cuda_twin().tba_synth_logits_host(out.ctypes.data, 0 if dtype == "bf16" else 1,
                                                     stream_key(seed, S_LOGITS), stream_key(seed, S_TOKENS),
                                                     stream_key(seed, S_PEAK), rows.ctypes.data, len(rows), V)
        if rc:
            raise RuntimeError(f"tba_synth_logits_host failed ({rc})")
    return out


def logits_rows_f64_host(seed: int, V: int, rows, dtype: str) -> np.ndarray:
    """``logits_rows_f64`` via the C host twin."""
    z = logits_rows_host(seed, V, rows, dtype)
    return bf16_bits_to_f64(z) if dtype == "bf16" else z.astype(np.float64)


# ----------------------------------------------------------------------------- TBA' inputs
S_GEN, S_GEN_OUT = 8, 9


def gen_logp(w: Workload, seed: int, seq0: int = 0, n: int | None = None) -> np.ndarray:
    """Per-token log-probs of the GENERATING policy pi_gen (TBA', Eq. 16: lambda_t =
    pi_theta/pi_gen), fp32 [n, T], 0 where masked. Modelled without any softmax: the stored
    logit of the sampled token minus the generator's expected log-partition (ln V + 2.65),
    plus U(-0.2, 0.2) policy drift, and on 2% of tokens a +-3 outlier (lambda ~ 20 or 0.05)
    so that IS clipping / IcePop masking are exercised."""
    n = w.N if n is None else n
    tok, mask = tokens_and_mask(w, seed, seq0, n)
    rows = (np.arange(seq0, seq0 + n, dtype=np.int64)[:, None] * w.T + np.arange(w.T)[None, :]).reshape(-1)
    y = raw_tokens(seed, w.V, rows.astype(np.uint64))
    h = hash64(seed, S_LOGITS, rows.astype(np.uint64) * np.uint64(w.V) + y.astype(np.uint64))
    acc = np.zeros(h.shape, dtype=np.int64)
    for k in range(4):
        acc += ((h >> np.uint64(16 * k)) & np.uint64(0xFFFF)).astype(np.int64)
    z = ((acc - 131070).astype(np.float64) * (2.0 ** -14)).astype(np.float32)
    z = (z + peak_of(seed, rows.astype(np.uint64))).astype(np.float32)
    if w.dtype == "bf16":
        z = bf16_bits_to_f64(f32_to_bf16_bits(z))
    u = unit24(hash64(seed, S_GEN, rows.astype(np.uint64)))
    out_sel = mulhi_u64(hash64(seed, S_GEN_OUT, rows.astype(np.uint64)), 100)
    drift = -0.2 + 0.4 * u
    drift = np.where(out_sel == 0, 3.0, np.where(out_sel == 1, -3.0, drift))
    g = (z.astype(np.float64) - (math.log(w.V) + 2.65) + drift).astype(np.float32).reshape(n, w.T)
    return np.where(mask == 1, g, np.float32(0.0)).astype(np.float32)


# ----------------------------------------------------------------------------- LM-head inputs (NEXT 3)
S_HIDDEN, S_WEIGHT = 10, 11


def weight_scale_exp(d: int) -> int:
    """Power-of-two exponent of the LM-head weight scale: logits z = W h then have a standard
    deviation of ~2.3 (the logits recipe's Irwin-Hall spread) for hidden states of std ~1.15."""
    return int(round(math.log2(0.866 / math.sqrt(d)))) - 14


def _bf16_matrix(seed: int, stream: int, d: int, rows, scale_exp: int, kind: str) -> np.ndarray:
    rows = np.asarray(rows, dtype=np.uint64).reshape(-1)
    idx = rows[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :]
    h = hash64(seed, stream, idx)
    if kind == "lattice":  # {-2, -1, 0, 1, 2} / 4: every partial sum of a dot product is exact in fp32
        x = (mulhi_u64(h, 5).astype(np.int64) - 2).astype(np.float64) * 0.25
    elif kind == "normal":  # Irwin-Hall(4) of the hash's 16-bit fields, times 2^scale_exp
        acc = np.zeros(h.shape, dtype=np.int64)
        for k in range(4):
            acc += ((h >> np.uint64(16 * k)) & np.uint64(0xFFFF)).astype(np.int64)
        x = (acc - 131070).astype(np.float64) * (2.0 ** scale_exp)
    else:
        raise ValueError(kind)
    return f32_to_bf16_bits(x.astype(np.float32))


def hidden_rows(seed: int, d: int, rows, kind: str = "normal") -> np.ndarray:
    """Final hidden states h_r (bf16 bits [len(rows), d]) of the given global rows."""
    return _bf16_matrix(seed, S_HIDDEN, d, rows, -15, kind)


def weight_rows(seed: int, d: int, vrows, kind: str = "normal") -> np.ndarray:
    """LM-head weight rows W_v (bf16 bits [len(vrows), d])."""
    return _bf16_matrix(seed, S_WEIGHT, d, vrows, weight_scale_exp(d), kind)


def fill_bf16_cuda(out, seed: int, which: str, row0: int, kind: str = "normal", stream: int | None = None):
    """Fill a CUDA bf16 tensor viewed as [nrows, d] (unit stride over d, rows uniformly strided)
    with hidden_rows / weight_rows of global rows row0..; bit-identical to the NumPy twin."""
    import torch
    if out.dtype != torch.bfloat16 or out.stride(-1) != 1:
        raise ValueError("out must be bf16 with unit stride over d")
    d = out.shape[-1]
    nrows = out.numel() // d if out.numel() else 0
    rs = out.stride(-2) if out.dim() >= 2 and out.shape[-2] > 1 else d
    stream_id, e = (S_HIDDEN, -15) if which == "hidden" else (S_WEIGHT, weight_scale_exp(d))
    s = torch.cuda.current_stream(out.device).cuda_stream if stream is None else stream
    L = _load_cuda_twin()
    rc = L.tba_synth_bf16(out.data_ptr(), stream_key(seed, stream_id), row0, nrows, d, rs,
                          1 if kind == "lattice" else 0, e, s)
    if rc:
        raise RuntimeError(f"tba_synth_bf16 failed ({rc})")
    return out
