"""The C ABI library loads without a GPU, exports every symbol include/tba.h declares, and
its host-side validation returns the documented status codes before touching CUDA."""
import ctypes
import math
import re
import os

import pytest

from paper_2503_18929_b200 import _lib
from paper_2503_18929_b200._lib import TbaRows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2503_18929_b200 import _build
    _build.build()
    return _lib.load()


def test_header_declarations_are_exported(L):
    hdr = open(os.path.join(ROOT, "include", "tba.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(tba_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name)
    # nm-level check: the .so really exports them with C linkage
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_synth_twin_exports():
    import tba_synth
    L2 = tba_synth._load_cuda_twin()
    assert hasattr(L2, "tba_synth_logits")


def test_version_and_strings(L):
    assert L.tba_abi_version() == 1
    for c in range(4):
        assert L.tba_status_string(c).startswith(b"TBA_")
    assert b"unknown" in L.tba_status_string(99)


def test_workspace_bytes(L):
    assert L.tba_workspace_bytes(0, 0) >= 256
    b = L.tba_workspace_bytes(64, 1024)
    assert b >= 64 * 1024 * 16 + 64 * 8
    assert L.tba_workspace_bytes(-1, 4) == 0


FAKE = 0x10000  # a non-null, aligned pointer value: validation must fail before any use


def _rows(**kw):
    d = dict(logits=FAKE, dtype=0, _pad=0, n_seq=8, seq_len=4, vocab=100, row_stride=100, tokens=FAKE, mask=FAKE)
    d.update(kw)
    return TbaRows(**d)


def _fwd(L, x, beta=1.0, K=4, ng=8.0, ptr=FAKE):
    return L.tba_vargrad_tb_loss_fwd(ctypes.byref(x), ptr, ptr, beta, K, ng, 0x100000, ptr, ptr, ptr, ptr, ptr,
                                     None, None)


def test_fwd_config_errors(L):
    x = _rows()
    for beta in (0.0, -1.0, math.nan, math.inf):
        assert _fwd(L, x, beta=beta) == _lib.TBA_ERR_INVALID_CONFIG
    for K in (1, 0, -3):
        assert _fwd(L, x, K=K) == _lib.TBA_ERR_INVALID_CONFIG


@pytest.mark.parametrize("kw", [dict(n_seq=-1), dict(seq_len=-2), dict(vocab=0), dict(row_stride=99),
                                dict(dtype=5), dict(logits=0), dict(tokens=0), dict(mask=0),
                                dict(logits=FAKE + 1), dict(dtype=1, logits=FAKE + 2), dict(tokens=FAKE + 4),
                                dict(n_seq=2 ** 40, seq_len=2 ** 30), dict(row_stride=2 ** 62),
                                dict(n_seq=2 ** 20, seq_len=2 ** 10)])
def test_rows_arg_errors(L, kw):
    x = _rows(**kw)
    assert _fwd(L, x) == _lib.TBA_ERR_INVALID_ARG
    assert L.tba_seq_logprob(ctypes.byref(x), 0x100000, FAKE, FAKE, None, None) == _lib.TBA_ERR_INVALID_ARG
    assert L.tba_vargrad_tb_loss_bwd(ctypes.byref(x), 0x100000, FAKE, 1.0, None, FAKE, 0, 100, None) == \
        _lib.TBA_ERR_INVALID_ARG


def test_fwd_arg_errors(L):
    assert _fwd(L, _rows(n_seq=6), K=4, ng=6.0) == _lib.TBA_ERR_INVALID_ARG      # N % K
    assert _fwd(L, _rows(), ng=4.0) == _lib.TBA_ERR_INVALID_ARG                  # N_global < N
    assert _fwd(L, _rows(), ng=math.nan) == _lib.TBA_ERR_INVALID_ARG
    assert _fwd(L, _rows(), ptr=0) == _lib.TBA_ERR_INVALID_ARG                   # null outputs
    assert L.tba_vargrad_tb_loss_fwd(ctypes.byref(_rows()), FAKE, FAKE, 1.0, 4, 8.0, 0x100010, FAKE, FAKE, FAKE,
                                     FAKE, FAKE, None, None) == _lib.TBA_ERR_INVALID_ARG  # misaligned workspace
    assert L.tba_vargrad_tb_loss_fwd(None, FAKE, FAKE, 1.0, 4, 8.0, 0x100000, FAKE, FAKE, FAKE, FAKE, FAKE, None,
                                     None) == _lib.TBA_ERR_INVALID_ARG


def test_bwd_arg_errors(L):
    x = _rows()
    bwd = lambda **k: L.tba_vargrad_tb_loss_bwd(ctypes.byref(x), k.get("ws", 0x100000), k.get("resid", FAKE),
                                               k.get("gs", 1.0), None, k.get("out", FAKE + 0x1000),
                                               k.get("dt", 0), k.get("ors", 100), None)
    assert bwd(dt=3) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(ors=99) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(gs=math.inf) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(out=0) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(resid=0) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(ws=0) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(out=FAKE + 1) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(out=FAKE, dt=1) == _lib.TBA_ERR_INVALID_ARG      # aliasing with a different dtype
    assert bwd(out=FAKE, ors=128) == _lib.TBA_ERR_INVALID_ARG   # aliasing with a different stride
    # partial overlap: dlogits starting two rows into the logits, or ending inside them
    rows = x.n_seq * x.seq_len
    assert bwd(out=FAKE + 2 * 100 * 2) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(out=FAKE - (rows - 1) * 100 * 2) == _lib.TBA_ERR_INVALID_ARG
    assert bwd(out=FAKE + 2, ors=100) == _lib.TBA_ERR_INVALID_ARG
    # disjoint ranges pass validation (then fail only at the launch on this GPU-less host)
    far = FAKE + rows * 100 * 2 + 0x10000
    assert bwd(out=far) != _lib.TBA_ERR_INVALID_ARG


def test_empty_batch_is_ok_without_gpu_work(L):
    # zero rows: seq_logprob has nothing to launch
    x = _rows(n_seq=0, logits=0, tokens=0, mask=0)
    assert L.tba_seq_logprob(ctypes.byref(x), 0, 0, 0, None, None) == _lib.TBA_OK
    assert L.tba_vargrad_tb_loss_bwd(ctypes.byref(x), 0, 0, 1.0, None, 0, 0, 100, None) == _lib.TBA_OK


def test_pipelined_validation(L):
    x = _rows()
    pipe = lambda xx, beta=1.0, K=4, ng=8.0, gs=0.25, ws=0x100000, out=FAKE + 0x1000, dt=0, ors=100: \
        L.tba_tb_loss_pipelined(ctypes.byref(xx) if xx is not None else None, None, FAKE, FAKE, beta, K, ng, gs, 0,
                                ws, FAKE, FAKE, FAKE, FAKE, FAKE, out, dt, ors, None, None, None, None)
    assert pipe(x, beta=0.0) == _lib.TBA_ERR_INVALID_CONFIG
    assert pipe(x, K=1) == _lib.TBA_ERR_INVALID_CONFIG
    assert pipe(_rows(n_seq=6), ng=6.0) == _lib.TBA_ERR_INVALID_ARG
    assert pipe(x, ng=4.0) == _lib.TBA_ERR_INVALID_ARG
    assert pipe(x, gs=math.nan) == _lib.TBA_ERR_INVALID_ARG
    assert pipe(x, dt=2) == _lib.TBA_ERR_INVALID_ARG
    assert pipe(x, ors=99) == _lib.TBA_ERR_INVALID_ARG
    assert pipe(x, ws=0x100010) == _lib.TBA_ERR_INVALID_ARG
    assert pipe(None) == _lib.TBA_ERR_INVALID_ARG


def _lm(**kw):
    d = dict(hidden=FAKE, weight=FAKE, n_seq=8, seq_len=4, d=64, vocab=100, hidden_stride=64, weight_stride=64,
             tokens=FAKE, mask=FAKE)
    d.update(kw)
    return _lib.TbaLmhead(**d)


@pytest.mark.parametrize("kw", [dict(d=12), dict(d=4), dict(hidden_stride=60), dict(hidden_stride=68),
                                dict(weight_stride=72 + 4), dict(hidden=FAKE + 8), dict(weight=FAKE + 2),
                                dict(hidden=0), dict(tokens=0), dict(mask=0), dict(vocab=0), dict(vocab=2 ** 31),
                                dict(n_seq=-1), dict(n_seq=2 ** 20, seq_len=2 ** 12), dict(tokens=FAKE + 4)])
def test_lmhead_validation(L, kw):
    x = _lm(**kw)
    assert L.tba_lmhead_seq_logprob(ctypes.byref(x), 1.0, 0x100000, FAKE, FAKE, None, None) == \
        _lib.TBA_ERR_INVALID_ARG
    assert L.tba_lmhead_tb_loss_fwd(ctypes.byref(x), None, FAKE, FAKE, 1.0, 4, 8.0, 0x100000, FAKE, FAKE, FAKE, FAKE,
                                    FAKE, None, None) == _lib.TBA_ERR_INVALID_ARG


def test_lmhead_config_and_workspace(L):
    x = _lm()
    assert L.tba_lmhead_seq_logprob(ctypes.byref(x), 0.0, 0x100000, FAKE, FAKE, None, None) == \
        _lib.TBA_ERR_INVALID_CONFIG
    assert L.tba_lmhead_tb_loss_fwd(ctypes.byref(x), None, FAKE, FAKE, -1.0, 4, 8.0, 0x100000, FAKE, FAKE, FAKE,
                                    FAKE, FAKE, None, None) == _lib.TBA_ERR_INVALID_CONFIG
    assert L.tba_lmhead_seq_logprob(ctypes.byref(x), 1.0, 0x100010, FAKE, FAKE, None, None) == \
        _lib.TBA_ERR_INVALID_ARG  # misaligned workspace
    base = L.tba_workspace_bytes(64, 1024)
    lm = L.tba_lmhead_workspace_bytes(64, 1024, 152064)
    assert lm >= base + 65536 * 149 * 8 + 65536 * 4   # per-(row, group of 1024) partials + gathered logit
    assert L.tba_lmhead_workspace_bytes(-1, 4, 10) == 0 and L.tba_lmhead_workspace_bytes(1, 4, 0) == 0
    empty = _lm(n_seq=0, hidden=0, weight=0, tokens=0, mask=0)
    assert L.tba_lmhead_seq_logprob(ctypes.byref(empty), 1.0, 0, 0, 0, None, None) == _lib.TBA_OK


def _lmb(L, x, opts=None, ws=0x100000, resid=FAKE, gs=0.25, dh=FAKE + 0x10000, dht=_lib.TBA_FP32, dhs=64,
         dw=FAKE + 0x20000, dws=64, acc=0, dlz=None, K=4, chunk=0, bws=0x200000):
    return L.tba_lmhead_tb_loss_bwd(ctypes.byref(x), opts, ws, resid, gs, None, dh, dht, dhs, dw, dws, acc, dlz, K,
                                    chunk, bws, None)


def test_lmhead_bwd_validation(L):
    x = _lm()
    bad = _lib.TBA_ERR_INVALID_ARG
    assert _lmb(L, _lm(d=12)) == bad
    assert _lmb(L, x, dht=7) == bad                       # unknown dhidden dtype
    assert _lmb(L, x, dhs=32) == bad                      # dhidden row stride < d
    assert _lmb(L, x, dh=FAKE + 2) == bad                 # misaligned fp32 dhidden
    assert _lmb(L, x, dh=FAKE) == bad                     # dhidden aliases hidden
    assert _lmb(L, x, dh=FAKE + 64) == bad                # dhidden overlaps hidden from its second element on
    assert _lmb(L, x, dws=63) == bad                      # dweight row stride < d
    assert _lmb(L, x, dw=FAKE + 0x20002) == bad           # misaligned dweight
    assert _lmb(L, x, bws=0x200010) == bad                # misaligned bwd workspace
    assert _lmb(L, x, bws=0) == bad                       # missing bwd workspace
    assert _lmb(L, x, ws=0x100008) == bad                 # misaligned forward workspace
    assert _lmb(L, x, resid=None) == bad
    assert _lmb(L, x, gs=math.inf) == bad
    assert _lmb(L, x, dlz=FAKE, K=3) == bad               # 8 sequences are not groups of 3
    opts = _lib.TbaTbOpts(0.0, None)
    assert _lmb(L, x, opts=ctypes.byref(opts)) == _lib.TBA_ERR_INVALID_CONFIG
    # nothing requested: OK without touching CUDA
    assert _lmb(L, x, dh=None, dw=None) == _lib.TBA_OK
    assert L.tba_lmhead_tbap_loss_bwd(ctypes.byref(x), 0x100000, None, -0.1, None, FAKE + 0x10000, _lib.TBA_FP32,
                                      64, None, 0, 0, 0, 0x200000, None) == bad  # no coef
    assert L.tba_lmhead_tbap_loss_bwd(ctypes.byref(x), 0x100000, FAKE + 2, -0.1, None, FAKE + 0x10000,
                                      _lib.TBA_FP32, 64, None, 0, 0, 0, 0x200000, None) == bad  # misaligned coef


def test_lmhead_bwd_workspace_bytes(L):
    rows, d, V, C = 65536, 3584, 152064, 16384
    b = L.tba_lmhead_bwd_workspace_bytes(64, 1024, d, V, C)
    # W^T, Hc, dZ, row list (dW reads dZ and Hc as MN-major operands: no transposed copies by default)
    need = d * V * 2 + C * d * 2 + C * V * 2 + rows * 4
    need += 4 * C * d * 4                                           # dH split-K partials (<= 4 fp32 slices)
    assert need <= b < need + 16 * 256
    # the chunk is rounded up to 128 rows and capped at the batch
    assert L.tba_lmhead_bwd_workspace_bytes(1, 100, 64, 1000, 0) == L.tba_lmhead_bwd_workspace_bytes(1, 100, 64, 1000, 128)
    assert L.tba_lmhead_bwd_workspace_bytes(1, 100, 64, 1000, 1) == L.tba_lmhead_bwd_workspace_bytes(1, 100, 64, 1000, 100)
    assert L.tba_lmhead_bwd_workspace_bytes(-1, 4, 64, 10, 0) == 0 and L.tba_lmhead_bwd_workspace_bytes(1, 4, 64, 0, 0) == 0


def test_lmhead_fwd_bwd_validation_and_workspace(L):
    x = _lm()

    def fb(x=x, beta=1.0, K=4, ng=8.0, gs=0.25, ws=0x100000, bws=0x200000, dh=FAKE + 0x10000, dht=_lib.TBA_FP32,
           dhs=64, partial=FAKE):
        return L.tba_lmhead_tb_loss_fwd_bwd(ctypes.byref(x), None, FAKE, FAKE, beta, K, ng, gs, 0, ws, FAKE, FAKE,
                                            FAKE, FAKE, partial, dh, dht, dhs, FAKE + 0x20000, 64, 0, None, bws,
                                            None, None)
    assert fb(beta=0.0) == _lib.TBA_ERR_INVALID_CONFIG
    assert fb(K=1) == _lib.TBA_ERR_INVALID_CONFIG
    assert fb(K=3) == _lib.TBA_ERR_INVALID_ARG          # 8 sequences are not groups of 3
    assert fb(ng=4.0) == _lib.TBA_ERR_INVALID_ARG       # n_seq_global < n_seq
    assert fb(gs=math.nan) == _lib.TBA_ERR_INVALID_ARG
    assert fb(partial=None) == _lib.TBA_ERR_INVALID_ARG
    assert fb(dh=FAKE) == _lib.TBA_ERR_INVALID_ARG      # dhidden aliases hidden
    assert fb(dht=5) == _lib.TBA_ERR_INVALID_ARG
    assert fb(dhs=8) == _lib.TBA_ERR_INVALID_ARG
    assert fb(ws=0x100004) == _lib.TBA_ERR_INVALID_ARG
    assert fb(bws=0) == _lib.TBA_ERR_INVALID_ARG
    assert fb(x=_lm(hidden_stride=60)) == _lib.TBA_ERR_INVALID_ARG
    # workspace: the stored fp32 logits of one chunk (2 Qwen groups = 16384 rows) dominate
    b = L.tba_lmhead_fwd_bwd_workspace_bytes(64, 1024, 3584, 152064, 8, 0)
    assert b >= 16384 * 152064 * 4 + 16384 * 152064 * 2
    # one group larger than the 16384-row GEMM chunk (Table 5: K = 16 x T = 2048 = 32768 rows): the
    # stored logits cover the group, every other backward buffer stays at the 16384-row chunk
    big = L.tba_lmhead_fwd_bwd_workspace_bytes(16, 2048, 3584, 152064, 16, 0)
    zst = 32768 * 152064 * 4
    assert zst < big < zst + 16384 * 152064 * 2 + 3584 * 152064 * 2 + 4 * 16384 * 3584 * 4 + 16384 * 3584 * 2 + \
        32768 * 152064 // 1024 * 16 + (1 << 24)
    assert L.tba_lmhead_fwd_bwd_workspace_bytes(64, 1024, 3584, 152064, 8, 1) < b   # one group per chunk
    assert L.tba_lmhead_fwd_bwd_workspace_bytes(9, 4, 64, 100, 4, 0) == 0          # 9 % 4 != 0
    assert L.tba_lmhead_fwd_bwd_workspace_bytes(0, 4, 64, 100, 4, 0) == 256
