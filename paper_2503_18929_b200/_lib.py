"""ctypes view of libtba.so (include/tba.h). Argument marshalling only.

The library is loaded from the package directory (in-tree build). If it is missing the
import of any op raises — there is no CPU or PyTorch fallback on the product path.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# TBA_LIBRARY: load an A/B build of the same library instead (developer switch, _build.build_variant)
LIB_PATH = os.environ.get("TBA_LIBRARY") or os.path.join(_HERE, "libtba.so")

TBA_OK, TBA_ERR_INVALID_ARG, TBA_ERR_INVALID_CONFIG, TBA_ERR_CUDA = 0, 1, 2, 3
TBA_DEV_TOKEN_RANGE, TBA_DEV_NONFINITE_ROW = 1, 2
TBA_BF16, TBA_FP32 = 0, 1

# every symbol include/tba.h declares (checked by tests/test_abi.py)
EXPORTS = ("tba_abi_version", "tba_status_string", "tba_workspace_bytes", "tba_seq_logprob", "tba_token_logprob",
           "tba_vargrad_tb_loss_fwd", "tba_vargrad_tb_loss_bwd", "tba_tb_loss_fwd", "tba_tb_loss_bwd", "tba_tb_loss_fused",
           "tba_tb_loss_pipelined", "tba_tb_loss_fwd_deferred",
           "tba_tbap_loss_fwd", "tba_tbap_loss_bwd", "tba_tbap_loss_fwd_deferred",
           "tba_lmhead_workspace_bytes", "tba_lmhead_seq_logprob", "tba_lmhead_tb_loss_fwd",
           "tba_lmhead_token_logprob", "tba_lmhead_tbap_loss_fwd", "tba_lmhead_bwd_workspace_bytes",
           "tba_lmhead_tb_loss_bwd", "tba_lmhead_tbap_loss_bwd", "tba_lmhead_fwd_bwd_workspace_bytes",
           "tba_lmhead_tb_loss_fwd_bwd")
TBA_IS_NONE, TBA_IS_CLIP, TBA_IS_ICEPOP = 0, 1, 2


class TbaRows(ctypes.Structure):
    _fields_ = [("logits", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("n_seq", ctypes.c_int64), ("seq_len", ctypes.c_int64), ("vocab", ctypes.c_int64),
                ("row_stride", ctypes.c_int64), ("tokens", ctypes.c_void_p), ("mask", ctypes.c_void_p)]


class TbaLmhead(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_void_p), ("weight", ctypes.c_void_p), ("n_seq", ctypes.c_int64),
                ("seq_len", ctypes.c_int64), ("d", ctypes.c_int64), ("vocab", ctypes.c_int64),
                ("hidden_stride", ctypes.c_int64), ("weight_stride", ctypes.c_int64), ("tokens", ctypes.c_void_p),
                ("mask", ctypes.c_void_p)]


class TbaTbOpts(ctypes.Structure):
    _fields_ = [("inv_temp", ctypes.c_double), ("log_z_param", ctypes.c_void_p)]


class TbaError(ValueError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {status_string(code)} (code {code})")


_lib = None
_lock = threading.Lock()


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libtba.so (once). Raises ImportError if the extension has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise ImportError(f"libtba.so not built at {p}: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(p)
        P, I32, I64, D, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
        RP = ctypes.POINTER(TbaRows)
        L.tba_abi_version.restype = ctypes.c_int
        L.tba_abi_version.argtypes = []
        L.tba_status_string.restype = ctypes.c_char_p
        L.tba_status_string.argtypes = [ctypes.c_int]
        L.tba_workspace_bytes.restype = SZ
        L.tba_workspace_bytes.argtypes = [I64, I64]
        L.tba_seq_logprob.restype = ctypes.c_int
        L.tba_seq_logprob.argtypes = [RP, P, P, P, P, P]
        L.tba_token_logprob.restype = ctypes.c_int
        L.tba_token_logprob.argtypes = [RP, D, P, P, P, P]
        L.tba_vargrad_tb_loss_fwd.restype = ctypes.c_int
        L.tba_vargrad_tb_loss_fwd.argtypes = [RP, P, P, D, I32, D, P, P, P, P, P, P, P, P]
        L.tba_vargrad_tb_loss_bwd.restype = ctypes.c_int
        L.tba_vargrad_tb_loss_bwd.argtypes = [RP, P, P, D, P, P, I32, I64, P]
        OP = ctypes.POINTER(TbaTbOpts)
        L.tba_tb_loss_fwd.restype = ctypes.c_int
        L.tba_tb_loss_fwd.argtypes = [RP, OP, P, P, D, I32, D, P, P, P, P, P, P, P, P]
        L.tba_tb_loss_bwd.restype = ctypes.c_int
        L.tba_tb_loss_bwd.argtypes = [RP, OP, P, P, D, P, P, I32, I64, P, I32, P]
        L.tba_tb_loss_fused.restype = ctypes.c_int
        L.tba_tb_loss_fused.argtypes = [RP, OP, P, P, D, I32, D, D, P, P, P, P, P, P, P, I32, I64, P, P, P]
        L.tba_tb_loss_pipelined.restype = ctypes.c_int
        L.tba_tb_loss_pipelined.argtypes = [RP, OP, P, P, D, I32, D, D, I32, P, P, P, P, P, P, P, I32, I64, P, P, P, P]
        L.tba_tb_loss_fwd_deferred.restype = ctypes.c_int
        L.tba_tb_loss_fwd_deferred.argtypes = [RP, OP, P, P, D, I32, D, P, P, P, P, P, P, P, I32, I64, P, P]
        LP = ctypes.POINTER(TbaLmhead)
        L.tba_lmhead_workspace_bytes.restype = SZ
        L.tba_lmhead_workspace_bytes.argtypes = [I64, I64, I64]
        L.tba_lmhead_seq_logprob.restype = ctypes.c_int
        L.tba_lmhead_seq_logprob.argtypes = [LP, D, P, P, P, P, P]
        L.tba_lmhead_tb_loss_fwd.restype = ctypes.c_int
        L.tba_lmhead_tb_loss_fwd.argtypes = [LP, OP, P, P, D, I32, D, P, P, P, P, P, P, P, P]
        L.tba_lmhead_token_logprob.restype = ctypes.c_int
        L.tba_lmhead_token_logprob.argtypes = [LP, D, P, P, P, P]
        L.tba_lmhead_tbap_loss_fwd.restype = ctypes.c_int
        L.tba_lmhead_tbap_loss_fwd.argtypes = [LP, P, P, P, D, I32, I32, D, D, D, P, P, P, P, P, P, P, P]
        L.tba_lmhead_bwd_workspace_bytes.restype = SZ
        L.tba_lmhead_bwd_workspace_bytes.argtypes = [I64, I64, I64, I64, I64]
        L.tba_lmhead_tb_loss_bwd.restype = ctypes.c_int
        L.tba_lmhead_tb_loss_bwd.argtypes = [LP, OP, P, P, D, P, P, I32, I64, P, I64, I32, P, I32, I64, P, P]
        L.tba_lmhead_tbap_loss_bwd.restype = ctypes.c_int
        L.tba_lmhead_tbap_loss_bwd.argtypes = [LP, P, P, D, P, P, I32, I64, P, I64, I32, I64, P, P]
        L.tba_lmhead_fwd_bwd_workspace_bytes.restype = SZ
        L.tba_lmhead_fwd_bwd_workspace_bytes.argtypes = [I64, I64, I64, I64, I32, I32]
        L.tba_lmhead_tb_loss_fwd_bwd.restype = ctypes.c_int
        L.tba_lmhead_tb_loss_fwd_bwd.argtypes = [LP, OP, P, P, D, I32, D, D, I32, P, P, P, P, P, P, P, I32, I64, P,
                                                 I64, I32, P, P, P, P]
        L.tba_tbap_loss_fwd.restype = ctypes.c_int
        L.tba_tbap_loss_fwd.argtypes = [RP, P, P, P, D, I32, I32, D, D, D, P, P, P, P, P, P, P, P]
        L.tba_tbap_loss_fwd_deferred.restype = ctypes.c_int
        L.tba_tbap_loss_fwd_deferred.argtypes = [RP, P, P, P, D, I32, I32, D, D, D, P, P, P, P, P, P, P, I32, I64, P, P]
        L.tba_tbap_loss_bwd.restype = ctypes.c_int
        L.tba_tbap_loss_bwd.argtypes = [RP, P, P, D, P, P, I32, I64, P]
        if L.tba_abi_version() != 1:
            raise ImportError("libtba.so ABI version mismatch")
        _lib = L
        return L


def status_string(code: int) -> str:
    return load().tba_status_string(code).decode()


def check(code: int, where: str):
    if code != TBA_OK:
        raise TbaError(code, where)
