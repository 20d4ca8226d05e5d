"""PyTorch-facing calls over libtba.so: argument marshalling only.

PyTorch supplies device memory, the current CUDA stream and (optionally) the process
group; every step of the loss head runs in libtba.so's kernels. Names follow the C ABI
(include/tba.h) and the paper's notation (Eqs. 4-5).
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from ._lib import TBA_BF16, TBA_FP32, TbaRows, check

_DT = {torch.bfloat16: TBA_BF16, torch.float32: TBA_FP32}
_CHECK = os.environ.get("TBA_CHECK", "0") == "1"


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def make_rows(logits: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor) -> TbaRows:
    """Describe [N, T, V] logits (any row stride >= V, unit element stride), [N, T] int64
    tokens and [N, T] uint8/bool mask as a tba_rows struct. Shape/dtype errors raise."""
    if logits.dim() != 3:
        raise ValueError("logits must be [N, T, V]")
    if logits.dtype not in _DT:
        raise ValueError(f"logits dtype {logits.dtype} unsupported (bf16 or fp32)")
    if not logits.is_cuda:
        raise ValueError("logits must be a CUDA tensor (there is no CPU path)")
    N, T, V = logits.shape
    if tokens.shape != (N, T) or mask.shape != (N, T):
        raise ValueError("tokens and mask must be [N, T]")
    if tokens.dtype != torch.int64 or not tokens.is_contiguous():
        raise ValueError("tokens must be contiguous int64")
    if mask.dtype == torch.bool:
        mask = mask.view(torch.uint8)
    if mask.dtype != torch.uint8 or not mask.is_contiguous():
        raise ValueError("mask must be contiguous uint8/bool")
    if tokens.device != logits.device or mask.device != logits.device:
        raise ValueError("logits, tokens and mask must be on the same device")
    if N * T > 0:
        if logits.stride(2) != 1:
            raise ValueError("logits must have unit stride over the vocabulary")
        rs = logits.stride(1) if T > 1 else (logits.stride(0) if N > 1 else V)
        if N > 1 and logits.stride(0) != T * rs:
            raise ValueError("logits rows must be uniformly strided ([N, T] must flatten to rows)")
        if rs < V:
            raise ValueError("logits rows overlap (row stride < V)")
    else:
        rs = V
    return TbaRows(logits.data_ptr(), _DT[logits.dtype], 0, N, T, V, rs, tokens.data_ptr(),
                   mask.data_ptr())


def workspace_bytes(n_seq: int, seq_len: int) -> int:
    return int(_lib.load().tba_workspace_bytes(n_seq, seq_len))


def _workspace(dev, N, T):
    return torch.empty(max(workspace_bytes(N, T), 256), dtype=torch.uint8, device=dev)


def _status(dev):
    return torch.zeros(1, dtype=torch.int32, device=dev)


def _raise_dev_status(st: torch.Tensor, where: str):
    v = int(st.item())
    if v:
        raise ValueError(f"{where}: device status {v} (1 = token out of range, 2 = non-finite row)")


def seq_logprob(logits, tokens, mask, *, check_status: bool = _CHECK):
    """log pi(y_s | x) and token counts per sequence (tba_seq_logprob).

    Returns (seq_logp fp64 [N], n_tokens int32 [N]). No autograd (use it for pi_ref)."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    N, T = tokens.shape
    dev = logits.device
    out = torch.empty(N, dtype=torch.float64, device=dev)
    ntok = torch.empty(N, dtype=torch.int32, device=dev)
    ws = _workspace(dev, N, T)
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        check(L.tba_seq_logprob(ctypes.byref(x), ws.data_ptr(), out.data_ptr(), ntok.data_ptr(), _ptr(st),
                                _stream(dev)), "tba_seq_logprob")
    if st is not None:
        _raise_dev_status(st, "tba_seq_logprob")
    return out, ntok


def token_logprob(logits, tokens, mask, *, inv_temp: float = 1.0, check_status: bool = _CHECK):
    """Per-token log softmax(inv_temp * z)[y] (tba_token_logprob), fp64 [N, T], 0 where masked."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    N, T = tokens.shape
    dev = logits.device
    out = torch.empty((N, T), dtype=torch.float64, device=dev)
    ws = _workspace(dev, N, T)
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        check(L.tba_token_logprob(ctypes.byref(x), float(inv_temp), ws.data_ptr(), out.data_ptr(), _ptr(st),
                                  _stream(dev)), "tba_token_logprob")
    if st is not None:
        _raise_dev_status(st, "tba_token_logprob")
    return out


class _Fwd:
    """Outputs of one tba_vargrad_tb_loss_fwd call (device tensors)."""

    def __init__(self, N, K, dev):
        self.seq_logp = torch.empty(N, dtype=torch.float64, device=dev)
        self.n_tokens = torch.empty(N, dtype=torch.int32, device=dev)
        self.log_z = torch.empty(max(N // K, 1), dtype=torch.float64, device=dev)[: N // K]
        self.resid = torch.empty(N, dtype=torch.float64, device=dev)
        self.partial = torch.empty(3, dtype=torch.float64, device=dev)


def _opts(inv_temp: float, log_z_param):
    if inv_temp == 1.0 and log_z_param is None:
        return None
    return _lib.TbaTbOpts(float(inv_temp), None if log_z_param is None else log_z_param.data_ptr())


def vargrad_fwd(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int, n_seq_global: float,
                workspace=None, out: _Fwd | None = None, check_status: bool = _CHECK, inv_temp: float = 1.0,
                log_z_param=None):
    """Raw TB forward (tba_tb_loss_fwd; tba_vargrad_tb_loss_fwd when inv_temp = 1 and no learned
    log Z). log_z_param: optional fp64 [N/K] learned log Z(x_i) (Eq. 3). Returns (_Fwd, workspace)."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    N, T = tokens.shape
    dev = logits.device
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    if log_z_param is not None and (log_z_param.shape != (N // K,) or log_z_param.dtype != torch.float64
                                    or not log_z_param.is_contiguous() or log_z_param.device != dev):
        raise ValueError("log_z_param must be a contiguous fp64 [N/K] tensor on the logits' device")
    o = out or _Fwd(N, K, dev)
    ws = workspace if workspace is not None else _workspace(dev, N, T)
    st = _status(dev) if check_status else None
    opts = _opts(inv_temp, log_z_param)
    with torch.cuda.device(dev):
        args = (ref_logp.data_ptr(), log_reward.data_ptr(), float(beta), int(K), float(n_seq_global), ws.data_ptr(),
                o.seq_logp.data_ptr(), o.n_tokens.data_ptr(), o.log_z.data_ptr() if N else None, o.resid.data_ptr(),
                o.partial.data_ptr(), _ptr(st), _stream(dev))
        if opts is None:
            check(L.tba_vargrad_tb_loss_fwd(ctypes.byref(x), *args), "tba_vargrad_tb_loss_fwd")
        else:
            check(L.tba_tb_loss_fwd(ctypes.byref(x), ctypes.byref(opts), *args), "tba_tb_loss_fwd")
    if st is not None:
        _raise_dev_status(st, "tba_vargrad_tb_loss_fwd")
    return o, ws


def vargrad_bwd(logits, tokens, mask, workspace, resid, grad_scale: float, grad_out=None, dlogits=None,
                dlogits_dtype=None, inv_temp: float = 1.0, log_z_param=None, K: int = 0):
    """Raw TB backward (tba_tb_loss_bwd). Returns dlogits, or (dlogits, d_log_z) when a learned
    log_z_param is given (then K is required)."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    dev = logits.device
    if dlogits is None:
        dt = dlogits_dtype or logits.dtype
        dlogits = torch.empty(logits.shape, dtype=dt, device=dev)
    if dlogits.shape != logits.shape or dlogits.dtype not in _DT or dlogits.stride(2) != 1:
        raise ValueError("dlogits must match logits' shape with unit vocab stride (bf16/fp32)")
    N, T, V = dlogits.shape
    ors = dlogits.stride(1) if T > 1 else (dlogits.stride(0) if N > 1 else V)
    if N > 1 and T > 0 and dlogits.stride(0) != T * ors:
        raise ValueError("dlogits rows must be uniformly strided")
    if grad_out is not None:
        grad_out = grad_out.to(device=dev, dtype=torch.float64).contiguous()
    opts = _opts(inv_temp, log_z_param)
    d_log_z = None
    if log_z_param is not None:
        if K < 2:
            raise ValueError("K is required with a learned log_z_param")
        d_log_z = torch.empty(N // K, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        if opts is None:
            check(L.tba_vargrad_tb_loss_bwd(ctypes.byref(x), workspace.data_ptr(), resid.data_ptr(),
                                            float(grad_scale), _ptr(grad_out), dlogits.data_ptr(), _DT[dlogits.dtype],
                                            max(ors, V), _stream(dev)), "tba_vargrad_tb_loss_bwd")
        else:
            check(L.tba_tb_loss_bwd(ctypes.byref(x), ctypes.byref(opts), workspace.data_ptr(), resid.data_ptr(),
                                    float(grad_scale), _ptr(grad_out), dlogits.data_ptr(), _DT[dlogits.dtype],
                                    max(ors, V), _ptr(d_log_z), int(K), _stream(dev)), "tba_tb_loss_bwd")
    return dlogits if d_log_z is None else (dlogits, d_log_z)


class VarGradTBLoss(torch.autograd.Function):
    """L = Eq. 5 (VarGrad log Z, Eq. 4) or Eq. 3 (learned log Z) over the (sharded) batch;
    backward writes dlogits in one fused pass (and dL/dlog Z for a learned log Z)."""

    @staticmethod
    def forward(ctx, logits, log_z_param, tokens, mask, ref_logp, log_reward, beta, K, n_global, group,
                dlogits_dtype, inv_temp, aux, overlap=False):
        lzp = None if log_z_param is None else log_z_param.detach().contiguous()
        o, ws = vargrad_fwd(logits, tokens, mask, ref_logp, log_reward, beta, K, n_global, inv_temp=inv_temp,
                            log_z_param=lzp)
        pending = None
        if group is not None:
            if overlap:  # side-stream all-reduce; the returned loss is this rank's share
                from .dist import allreduce_partial_async
                pending = allreduce_partial_async(o.partial, group)
            else:
                import torch.distributed as dist
                dist.all_reduce(o.partial, op=dist.ReduceOp.SUM, group=group)
        ctx.save_for_backward(logits, tokens, mask, ws, o.resid)
        ctx.n_global, ctx.K, ctx.inv_temp = n_global, K, inv_temp
        ctx.dlogits_dtype = dlogits_dtype
        ctx.lzp = lzp
        if aux is not None:
            aux.update(seq_logp=o.seq_logp, n_tokens=o.n_tokens, log_z=o.log_z, resid=o.resid, partial=o.partial)
            if pending is not None:
                aux["global_partial"] = pending
        return o.partial[0]

    @staticmethod
    def backward(ctx, grad):
        logits, tokens, mask, ws, resid = ctx.saved_tensors
        r = vargrad_bwd(logits, tokens, mask, ws, resid, 2.0 / ctx.n_global, grad_out=grad,
                        dlogits_dtype=ctx.dlogits_dtype, inv_temp=ctx.inv_temp, log_z_param=ctx.lzp, K=ctx.K)
        d, dz = (r, None) if ctx.lzp is None else r
        return (d, dz) + (None,) * 12


def vargrad_tb_loss(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int, *, n_seq_global=None,
                    group=None, dlogits_dtype=None, return_aux: bool = False, log_z=None, inv_temp: float = 1.0,
                    overlap_allreduce: bool = False):
    """The trajectory-balance loss, autograd-enabled.

    Default: the VarGrad loss of Eq. 5 with the detached K-sample log Z of Eq. 4.
    ``log_z`` (fp64 [N/K] tensor, may require grad): a learned log Z(x_i) instead (Eq. 3,
    P:114-117). ``inv_temp``: log pi = log softmax(inv_temp * z).
    logits [N, T, V] bf16/fp32 (N = groups*K, group-major); tokens int64 [N, T]; mask
    uint8/bool [N, T]; ref_logp, log_reward fp64 [N] (log_reward is r_phi). With ``group``
    each rank passes its own whole groups and the partial sums are all-reduced once;
    ``n_seq_global`` defaults to N * world. With ``overlap_allreduce`` the all-reduce runs on a side
    stream and the returned (differentiable) loss is this rank's share sum_own eps^2 / N_global —
    whose gradient is exactly the global loss's, since L = sum over ranks of the shares — while
    ``aux["global_partial"].wait()`` gives the global [L, N_global, B_global]; the backward never
    waits for the collective (N_global is static). Returns the 0-dim fp64
    loss (and an aux dict with seq_logp, n_tokens, log_z, resid, partial when ``return_aux``)."""
    N = tokens.shape[0]
    if n_seq_global is None:
        if group is not None:
            import torch.distributed as dist
            n_seq_global = N * dist.get_world_size(group)
        else:
            n_seq_global = N
    aux = {} if return_aux else None
    loss = VarGradTBLoss.apply(logits, log_z, tokens, mask, ref_logp, log_reward, float(beta), int(K),
                               float(n_seq_global), group, dlogits_dtype, float(inv_temp), aux,
                               bool(overlap_allreduce))
    return (loss, aux) if return_aux else loss


_AUX_STREAMS: dict = {}


def _aux_stream(dev: torch.device) -> int:
    """A second stream per device for the pipelined schedule (created once, reused)."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _AUX_STREAMS:
        _AUX_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _AUX_STREAMS[key].cuda_stream


def _fwd_bwd_one_call(entry: str, logits, tokens, mask, ref_logp, log_reward, beta, K, n_seq_global, grad_scale,
                      workspace, out, dlogits, dlogits_dtype, inv_temp, log_z_param, check_status, extra_mid=(),
                      extra_tail=()):
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    N, T = tokens.shape
    dev = logits.device
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    if dlogits is None:
        dlogits = torch.empty(logits.shape, dtype=dlogits_dtype or logits.dtype, device=dev)
    Nn, Tt, V = dlogits.shape
    ors = dlogits.stride(1) if Tt > 1 else (dlogits.stride(0) if Nn > 1 else V)
    o = out or _Fwd(N, K, dev)
    ws = workspace if workspace is not None else _workspace(dev, N, T)
    st = _status(dev) if check_status else None
    d_log_z = torch.empty(N // K, dtype=torch.float64, device=dev) if log_z_param is not None else None
    opts = _opts(inv_temp, log_z_param)
    gs = 2.0 / float(n_seq_global) if grad_scale is None else float(grad_scale)
    with torch.cuda.device(dev):
        check(getattr(L, entry)(ctypes.byref(x), ctypes.byref(opts) if opts is not None else None,
                                ref_logp.data_ptr(), log_reward.data_ptr(), float(beta), int(K), float(n_seq_global),
                                gs, *extra_mid, ws.data_ptr(), o.seq_logp.data_ptr(), o.n_tokens.data_ptr(),
                                o.log_z.data_ptr() if N else None, o.resid.data_ptr(), o.partial.data_ptr(),
                                dlogits.data_ptr(), _DT[dlogits.dtype], max(ors, V), _ptr(d_log_z), _ptr(st),
                                _stream(dev), *extra_tail), entry)
    if st is not None:
        _raise_dev_status(st, entry)
    return o, ws, dlogits, d_log_z


def vargrad_fused(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int, n_seq_global: float,
                  grad_scale: float | None = None, workspace=None, out: _Fwd | None = None, dlogits=None,
                  dlogits_dtype=None, inv_temp: float = 1.0, log_z_param=None, check_status: bool = _CHECK):
    """One-launch forward + backward (tba_tb_loss_fused). grad_scale defaults to 2/n_seq_global
    (d loss / d logits with grad_out = 1). Returns (_Fwd, workspace, dlogits, d_log_z or None)."""
    return _fwd_bwd_one_call("tba_tb_loss_fused", logits, tokens, mask, ref_logp, log_reward, beta, K, n_seq_global,
                             grad_scale, workspace, out, dlogits, dlogits_dtype, inv_temp, log_z_param, check_status)


def vargrad_pipelined(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int, n_seq_global: float,
                      grad_scale: float | None = None, workspace=None, out: _Fwd | None = None, dlogits=None,
                      dlogits_dtype=None, inv_temp: float = 1.0, log_z_param=None, groups_per_chunk: int = 0,
                      aux_stream: bool = True, check_status: bool = _CHECK):
    """Forward + backward in group chunks on two streams (tba_tb_loss_pipelined): the gradient
    writer of chunk c-1 runs beside the forward of chunk c, so small groups are re-read from L2.
    Same results as vargrad_fwd + vargrad_bwd, bitwise. groups_per_chunk <= 0 picks ~L2/4 of
    logits per chunk. Returns (_Fwd, workspace, dlogits, d_log_z or None)."""
    dev = logits.device
    aux = _aux_stream(dev) if aux_stream else _stream(dev)
    return _fwd_bwd_one_call("tba_tb_loss_pipelined", logits, tokens, mask, ref_logp, log_reward, beta, K,
                             n_seq_global, grad_scale, workspace, out, dlogits, dlogits_dtype, inv_temp, log_z_param,
                             check_status, extra_mid=(int(groups_per_chunk),), extra_tail=(aux,))


def vargrad_fwd_deferred(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int, n_seq_global: float,
                         workspace=None, out: _Fwd | None = None, grad_unscaled=None, g_dtype=None,
                         inv_temp: float = 1.0, log_z_param=None, check_status: bool = _CHECK):
    """Deferred-scale forward (tba_tb_loss_fwd_deferred): the forward outputs plus the unscaled
    gradient G = mu * inv_temp * (onehot - softmax), written in the same pass; the true
    dlogits are (2 g / n_seq_global) * resid[s] * G (apply as a row scale downstream).
    Returns (_Fwd, workspace, G)."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    N, T = tokens.shape
    dev = logits.device
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    if grad_unscaled is None:
        grad_unscaled = torch.empty(logits.shape, dtype=g_dtype or logits.dtype, device=dev)
    Nn, Tt, V = grad_unscaled.shape
    ors = grad_unscaled.stride(1) if Tt > 1 else (grad_unscaled.stride(0) if Nn > 1 else V)
    o = out or _Fwd(N, K, dev)
    ws = workspace if workspace is not None else _workspace(dev, N, T)
    st = _status(dev) if check_status else None
    opts = _opts(inv_temp, log_z_param)
    with torch.cuda.device(dev):
        check(L.tba_tb_loss_fwd_deferred(ctypes.byref(x), ctypes.byref(opts) if opts is not None else None,
                                         ref_logp.data_ptr(), log_reward.data_ptr(), float(beta), int(K),
                                         float(n_seq_global), ws.data_ptr(), o.seq_logp.data_ptr(),
                                         o.n_tokens.data_ptr(), o.log_z.data_ptr() if N else None,
                                         o.resid.data_ptr(), o.partial.data_ptr(), grad_unscaled.data_ptr(),
                                         _DT[grad_unscaled.dtype], max(ors, V), _ptr(st), _stream(dev)),
              "tba_tb_loss_fwd_deferred")
    if st is not None:
        _raise_dev_status(st, "tba_tb_loss_fwd_deferred")
    return o, ws, grad_unscaled


def vargrad_tb_loss_and_grad(logits, tokens, mask, ref_logp, log_reward, beta: float, K: int, *, n_seq_global=None,
                             group=None, dlogits=None, dlogits_dtype=None, inv_temp: float = 1.0, log_z=None,
                             return_aux: bool = False, schedule: str = "fused"):
    """Loss AND d loss / d logits in one launch (no autograd): returns (loss, dlogits) or
    (loss, dlogits, d_log_z) with a learned log_z; aux dict appended when return_aux. The
    gradient is that of the (all-reduced, when `group` is given) batch loss of Eq. 5 / Eq. 3."""
    N = tokens.shape[0]
    if n_seq_global is None:
        if group is not None:
            import torch.distributed as dist
            n_seq_global = N * dist.get_world_size(group)
        else:
            n_seq_global = N
    if schedule not in ("fused", "pipelined"):
        raise ValueError("schedule must be 'fused' or 'pipelined'")
    call = vargrad_fused if schedule == "fused" else vargrad_pipelined
    o, ws, d, dz = call(logits, tokens, mask, ref_logp, log_reward, beta, K, float(n_seq_global),
                        dlogits=dlogits, dlogits_dtype=dlogits_dtype, inv_temp=inv_temp,
                        log_z_param=None if log_z is None else log_z.detach().contiguous())
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(o.partial, op=dist.ReduceOp.SUM, group=group)
    res = (o.partial[0], d) + ((dz,) if log_z is not None else ())
    if return_aux:
        res = res + (dict(seq_logp=o.seq_logp, n_tokens=o.n_tokens, log_z=o.log_z, resid=o.resid, partial=o.partial),)
    return res


# ----------------------------------------------------------------------------- LM-head-fused (NEXT 3)
def make_lmhead(hidden: torch.Tensor, weight: torch.Tensor, tokens: torch.Tensor, mask: torch.Tensor):
    """Describe [N, T, d] bf16 hidden states and a [V, d] bf16 LM-head weight as tba_lmhead."""
    if hidden.dim() != 3 or weight.dim() != 2:
        raise ValueError("hidden must be [N, T, d] and weight [V, d]")
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise ValueError("hidden and weight must be bf16")
    if not (hidden.is_cuda and weight.is_cuda) or hidden.device != weight.device:
        raise ValueError("hidden and weight must be CUDA tensors on one device (there is no CPU path)")
    N, T, d = hidden.shape
    V, d2 = weight.shape
    if d2 != d:
        raise ValueError("hidden and weight disagree on d")
    if tokens.shape != (N, T) or mask.shape != (N, T) or tokens.dtype != torch.int64 or not tokens.is_contiguous():
        raise ValueError("tokens must be contiguous int64 [N, T] and mask [N, T]")
    if mask.dtype == torch.bool:
        mask = mask.view(torch.uint8)
    if mask.dtype != torch.uint8 or not mask.is_contiguous():
        raise ValueError("mask must be contiguous uint8/bool")
    if hidden.stride(2) != 1 or weight.stride(1) != 1:
        raise ValueError("hidden and weight need unit stride over d")
    hs = hidden.stride(1) if T > 1 else (hidden.stride(0) if N > 1 else d)
    if N > 1 and T > 0 and hidden.stride(0) != T * hs:
        raise ValueError("hidden rows must be uniformly strided")
    ws_ = weight.stride(0) if V > 1 else d
    return _lib.TbaLmhead(hidden.data_ptr(), weight.data_ptr(), N, T, d, V, max(hs, d), max(ws_, d),
                          tokens.data_ptr(), mask.data_ptr())


def lmhead_workspace_bytes(n_seq: int, seq_len: int, vocab: int) -> int:
    return int(_lib.load().tba_lmhead_workspace_bytes(int(n_seq), int(seq_len), int(vocab)))


def _lm_workspace(dev, N, T, V):
    return torch.empty(max(lmhead_workspace_bytes(N, T, V), 256), dtype=torch.uint8, device=dev)


def lmhead_seq_logprob(hidden, weight, tokens, mask, *, inv_temp: float = 1.0, workspace=None,
                       check_status: bool = _CHECK):
    """log pi(y_s|x) from hidden states and the LM-head weight, logits never written
    (tba_lmhead_seq_logprob). Returns (seq_logp fp64 [N], n_tokens int32 [N])."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T = tokens.shape
    dev = hidden.device
    out = torch.empty(N, dtype=torch.float64, device=dev)
    ntok = torch.empty(N, dtype=torch.int32, device=dev)
    ws = workspace if workspace is not None else _lm_workspace(dev, N, T, weight.shape[0])
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        check(L.tba_lmhead_seq_logprob(ctypes.byref(x), float(inv_temp), ws.data_ptr(), out.data_ptr(),
                                       ntok.data_ptr(), _ptr(st), _stream(dev)), "tba_lmhead_seq_logprob")
    if st is not None:
        _raise_dev_status(st, "tba_lmhead_seq_logprob")
    return out, ntok


def lmhead_vargrad_fwd(hidden, weight, tokens, mask, ref_logp, log_reward, beta: float, K: int,
                       n_seq_global: float, *, inv_temp: float = 1.0, log_z_param=None, workspace=None,
                       out: _Fwd | None = None, check_status: bool = _CHECK):
    """VarGrad TB forward (Eqs. 4-5; Eq. 3 with log_z_param) from hidden states
    (tba_lmhead_tb_loss_fwd). Returns (_Fwd, workspace)."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T = tokens.shape
    dev = hidden.device
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    o = out or _Fwd(N, K, dev)
    ws = workspace if workspace is not None else _lm_workspace(dev, N, T, weight.shape[0])
    st = _status(dev) if check_status else None
    opts = _opts(inv_temp, log_z_param)
    with torch.cuda.device(dev):
        check(L.tba_lmhead_tb_loss_fwd(ctypes.byref(x), ctypes.byref(opts) if opts is not None else None,
                                       ref_logp.data_ptr(), log_reward.data_ptr(), float(beta), int(K),
                                       float(n_seq_global), ws.data_ptr(), o.seq_logp.data_ptr(),
                                       o.n_tokens.data_ptr(), o.log_z.data_ptr() if N else None,
                                       o.resid.data_ptr(), o.partial.data_ptr(), _ptr(st), _stream(dev)),
              "tba_lmhead_tb_loss_fwd")
    if st is not None:
        _raise_dev_status(st, "tba_lmhead_tb_loss_fwd")
    return o, ws


def lmhead_token_logprob(hidden, weight, tokens, mask, *, inv_temp: float = 1.0, workspace=None,
                         check_status: bool = _CHECK):
    """Per-token log-probs (fp64 [N, T], 0 where masked) from hidden states
    (tba_lmhead_token_logprob), logits never written."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T = tokens.shape
    dev = hidden.device
    out = torch.empty((N, T), dtype=torch.float64, device=dev)
    ws = workspace if workspace is not None else _lm_workspace(dev, N, T, weight.shape[0])
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        check(L.tba_lmhead_token_logprob(ctypes.byref(x), float(inv_temp), ws.data_ptr(), out.data_ptr(), _ptr(st),
                                         _stream(dev)), "tba_lmhead_token_logprob")
    if st is not None:
        _raise_dev_status(st, "tba_lmhead_token_logprob")
    return out


# ----------------------------------------------------------------------------- LM-head backward
def lmhead_bwd_workspace_bytes(n_seq: int, seq_len: int, d: int, vocab: int, chunk_rows: int = 0) -> int:
    return int(_lib.load().tba_lmhead_bwd_workspace_bytes(int(n_seq), int(seq_len), int(d), int(vocab),
                                                          int(chunk_rows)))


def _lm_grad_bufs(hidden, weight, dhidden, dweight, dhidden_dtype, want_dh, want_dw):
    dev = hidden.device
    if want_dh and dhidden is None:
        dhidden = torch.empty(hidden.shape, dtype=dhidden_dtype or torch.float32, device=dev)
    if want_dw and dweight is None:
        dweight = torch.empty(weight.shape, dtype=torch.float32, device=dev)
    dh_args = (None, 0, 0)
    if dhidden is not None:
        if dhidden.shape != hidden.shape or dhidden.dtype not in _DT or dhidden.stride(2) != 1 or \
                not dhidden.is_contiguous():
            raise ValueError("dhidden must be a contiguous bf16/fp32 tensor shaped like hidden")
        dh_args = (dhidden.data_ptr(), _DT[dhidden.dtype], hidden.shape[2])
    dw_args = (None, 0)
    if dweight is not None:
        if dweight.shape != weight.shape or dweight.dtype != torch.float32 or not dweight.is_contiguous():
            raise ValueError("dweight must be a contiguous fp32 tensor shaped like weight")
        dw_args = (dweight.data_ptr(), weight.shape[1])
    return dhidden, dweight, dh_args, dw_args


def _lm_bwd_ws(dev, N, T, d, V, chunk_rows):
    return torch.empty(max(lmhead_bwd_workspace_bytes(N, T, d, V, chunk_rows), 256), dtype=torch.uint8, device=dev)


def lmhead_vargrad_bwd(hidden, weight, tokens, mask, workspace, resid, grad_scale: float, *, grad_out=None,
                       inv_temp: float = 1.0, log_z_param=None, K: int = 0, dhidden=None, dweight=None,
                       dhidden_dtype=None, want_dhidden: bool = True, want_dweight: bool = True,
                       accumulate: bool = False, chunk_rows: int = 0, bwd_workspace=None):
    """Backward of the TB loss through the LM head (tba_lmhead_tb_loss_bwd): dL/dhidden ([N, T, d],
    fp32 unless dhidden_dtype=bf16) and dL/dW (fp32 [V, d]); the logits are recomputed on the tensor
    cores from the forward's `workspace`. Returns (dhidden, dweight[, d_log_z])."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T, d = hidden.shape
    dev = hidden.device
    dhidden, dweight, (dhp, dht, dhs), (dwp, dws) = _lm_grad_bufs(hidden, weight, dhidden, dweight, dhidden_dtype,
                                                                  want_dhidden, want_dweight)
    if grad_out is not None:
        grad_out = grad_out.to(device=dev, dtype=torch.float64).contiguous()
    opts = _opts(inv_temp, log_z_param)
    d_log_z = None
    if log_z_param is not None:
        if K < 2:
            raise ValueError("K is required with a learned log_z_param")
        d_log_z = torch.empty(N // K, dtype=torch.float64, device=dev)
    bws = bwd_workspace if bwd_workspace is not None else _lm_bwd_ws(dev, N, T, d, weight.shape[0], chunk_rows)
    with torch.cuda.device(dev):
        check(L.tba_lmhead_tb_loss_bwd(ctypes.byref(x), ctypes.byref(opts) if opts is not None else None,
                                       workspace.data_ptr(), resid.data_ptr(), float(grad_scale), _ptr(grad_out),
                                       dhp, dht, dhs, dwp, dws, int(bool(accumulate)), _ptr(d_log_z), int(K),
                                       int(chunk_rows), bws.data_ptr(), _stream(dev)), "tba_lmhead_tb_loss_bwd")
    return (dhidden, dweight) if d_log_z is None else (dhidden, dweight, d_log_z)


def lmhead_tbap_bwd(hidden, weight, tokens, mask, workspace, coef, n_tok_global: float, *, grad_out=None,
                    dhidden=None, dweight=None, dhidden_dtype=None, want_dhidden: bool = True,
                    want_dweight: bool = True, accumulate: bool = False, chunk_rows: int = 0, bwd_workspace=None):
    """Backward of the TBA' surrogate (Eq. 16) through the LM head (tba_lmhead_tbap_loss_bwd);
    grad_scale = -1 / n_tok_global. Returns (dhidden, dweight)."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T, d = hidden.shape
    dev = hidden.device
    dhidden, dweight, (dhp, dht, dhs), (dwp, dws) = _lm_grad_bufs(hidden, weight, dhidden, dweight, dhidden_dtype,
                                                                  want_dhidden, want_dweight)
    if grad_out is not None:
        grad_out = grad_out.to(device=dev, dtype=torch.float64).contiguous()
    bws = bwd_workspace if bwd_workspace is not None else _lm_bwd_ws(dev, N, T, d, weight.shape[0], chunk_rows)
    with torch.cuda.device(dev):
        check(L.tba_lmhead_tbap_loss_bwd(ctypes.byref(x), workspace.data_ptr(), coef.data_ptr(),
                                         -1.0 / float(n_tok_global), _ptr(grad_out), dhp, dht, dhs, dwp, dws,
                                         int(bool(accumulate)), int(chunk_rows), bws.data_ptr(), _stream(dev)),
              "tba_lmhead_tbap_loss_bwd")
    return dhidden, dweight


def lmhead_fwd_bwd_workspace_bytes(n_seq: int, seq_len: int, d: int, vocab: int, K: int,
                                   groups_per_chunk: int = 0) -> int:
    return int(_lib.load().tba_lmhead_fwd_bwd_workspace_bytes(int(n_seq), int(seq_len), int(d), int(vocab), int(K),
                                                              int(groups_per_chunk)))


def lmhead_vargrad_fwd_bwd(hidden, weight, tokens, mask, ref_logp, log_reward, beta: float, K: int,
                           n_seq_global: float, *, grad_out: float = 1.0, inv_temp: float = 1.0, log_z_param=None,
                           dhidden=None, dweight=None, dhidden_dtype=None, want_dhidden: bool = True,
                           want_dweight: bool = True, accumulate: bool = False, groups_per_chunk: int = 0,
                           workspace=None, bwd_workspace=None, out: _Fwd | None = None,
                           check_status: bool = _CHECK):
    """TB loss and its gradient through the LM head in one call (tba_lmhead_tb_loss_fwd_bwd): chunks of
    whole groups, the chunk's logits stored once in fp32 and reused by the gradient pass.
    grad_out (host float) scales the gradient: grad_scale = 2 grad_out / n_seq_global.
    Returns (_Fwd, dhidden, dweight[, d_log_z])."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T, d = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    dhidden, dweight, (dhp, dht, dhs), (dwp, dws) = _lm_grad_bufs(hidden, weight, dhidden, dweight, dhidden_dtype,
                                                                  want_dhidden, want_dweight)
    o = out or _Fwd(N, K, dev)
    ws = workspace if workspace is not None else _lm_workspace(dev, N, T, V)
    if bwd_workspace is None:
        bwd_workspace = torch.empty(max(lmhead_fwd_bwd_workspace_bytes(N, T, d, V, K, groups_per_chunk), 256),
                                    dtype=torch.uint8, device=dev)
    opts = _opts(inv_temp, log_z_param)
    d_log_z = torch.empty(N // K, dtype=torch.float64, device=dev) if log_z_param is not None else None
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        check(L.tba_lmhead_tb_loss_fwd_bwd(ctypes.byref(x), ctypes.byref(opts) if opts is not None else None,
                                           ref_logp.data_ptr(), log_reward.data_ptr(), float(beta), int(K),
                                           float(n_seq_global), 2.0 * float(grad_out) / float(n_seq_global),
                                           int(groups_per_chunk), ws.data_ptr(), o.seq_logp.data_ptr(),
                                           o.n_tokens.data_ptr(), o.log_z.data_ptr() if N else None,
                                           o.resid.data_ptr(), o.partial.data_ptr(), dhp, dht, dhs, dwp, dws,
                                           int(bool(accumulate)), _ptr(d_log_z), bwd_workspace.data_ptr(), _ptr(st),
                                           _stream(dev)), "tba_lmhead_tb_loss_fwd_bwd")
    if st is not None:
        _raise_dev_status(st, "tba_lmhead_tb_loss_fwd_bwd")
    return (o, dhidden, dweight) if d_log_z is None else (o, dhidden, dweight, d_log_z)


class LmHeadTBLoss(torch.autograd.Function):
    """Eq. 5 (or Eq. 3 with a learned log Z) from hidden states through the LM head, logits never
    materialised: forward tba_lmhead_tb_loss_fwd, backward tba_lmhead_tb_loss_bwd (dhidden, dW)."""

    @staticmethod
    def forward(ctx, hidden, weight, log_z_param, tokens, mask, ref_logp, log_reward, beta, K, n_global, group,
                inv_temp, chunk_rows, aux):
        lzp = None if log_z_param is None else log_z_param.detach().contiguous()
        o, ws = lmhead_vargrad_fwd(hidden, weight, tokens, mask, ref_logp, log_reward, beta, K, n_global,
                                   inv_temp=inv_temp, log_z_param=lzp)
        if group is not None:
            import torch.distributed as dist
            dist.all_reduce(o.partial, op=dist.ReduceOp.SUM, group=group)
        ctx.save_for_backward(hidden, weight, tokens, mask, ws, o.resid)
        ctx.n_global, ctx.K, ctx.inv_temp, ctx.lzp, ctx.chunk_rows = n_global, K, inv_temp, lzp, chunk_rows
        if aux is not None:
            aux.update(seq_logp=o.seq_logp, n_tokens=o.n_tokens, log_z=o.log_z, resid=o.resid, partial=o.partial)
            if pending is not None:
                aux["global_partial"] = pending
        return o.partial[0]

    @staticmethod
    def backward(ctx, grad):
        hidden, weight, tokens, mask, ws, resid = ctx.saved_tensors
        r = lmhead_vargrad_bwd(hidden, weight, tokens, mask, ws, resid, 2.0 / ctx.n_global, grad_out=grad,
                               inv_temp=ctx.inv_temp, log_z_param=ctx.lzp, K=ctx.K,
                               dhidden_dtype=hidden.dtype if hidden.dtype == torch.float32 else torch.float32,
                               want_dhidden=ctx.needs_input_grad[0], want_dweight=ctx.needs_input_grad[1],
                               chunk_rows=ctx.chunk_rows)
        dh, dw = r[0], r[1]
        dz = r[2] if ctx.lzp is not None else None
        return (dh.to(hidden.dtype) if dh is not None else None, dw.to(weight.dtype) if dw is not None else None,
                dz) + (None,) * 11


def lmhead_tb_loss(hidden, weight, tokens, mask, ref_logp, log_reward, beta: float, K: int, *, n_seq_global=None,
                   group=None, log_z=None, inv_temp: float = 1.0, chunk_rows: int = 0, return_aux: bool = False):
    """The trajectory-balance loss from final hidden states [N, T, d] (bf16) and the LM-head weight
    [V, d] (bf16), autograd-enabled for hidden, weight and a learned log_z; z = W h is never written
    to memory in either direction. Arguments otherwise as vargrad_tb_loss."""
    N = tokens.shape[0]
    if n_seq_global is None:
        if group is not None:
            import torch.distributed as dist
            n_seq_global = N * dist.get_world_size(group)
        else:
            n_seq_global = N
    aux = {} if return_aux else None
    loss = LmHeadTBLoss.apply(hidden, weight, log_z, tokens, mask, ref_logp, log_reward, float(beta), int(K),
                              float(n_seq_global), group, float(inv_temp), int(chunk_rows), aux)
    return (loss, aux) if return_aux else loss


# ----------------------------------------------------------------------------- TBA' (Eq. 16)
_IS = {"none": 0, "clip": 1, "icepop": 2}


class _TbapFwd:
    """Outputs of one tba_tbap_loss_fwd call (device tensors)."""

    def __init__(self, N, T, dev):
        self.seq_logp = torch.empty(N, dtype=torch.float64, device=dev)
        self.n_tokens = torch.empty(N, dtype=torch.int32, device=dev)
        self.adv = torch.empty(N, dtype=torch.float64, device=dev)
        self.coef = torch.empty((N, T), dtype=torch.float32, device=dev)
        self.partial = torch.empty(3, dtype=torch.float64, device=dev)


def tbap_fwd(logits, tokens, mask, gen_logp, ref_logp, log_reward, beta: float, K: int, is_mode: str = "clip",
             is_lo: float = 0.0, is_hi: float = 8.0, n_tok_global: float | None = None, workspace=None,
             out: _TbapFwd | None = None, check_status: bool = _CHECK, grad_unscaled=None):
    """Raw TBA' forward (tba_tbap_loss_fwd, Eq. 16). gen_logp: fp32 [N, T] log-probs of the
    generating policy. n_tok_global defaults to this call's valid-token count (host sync)."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    N, T = tokens.shape
    dev = logits.device
    if gen_logp.shape != (N, T) or gen_logp.dtype != torch.float32 or not gen_logp.is_contiguous():
        raise ValueError("gen_logp must be a contiguous fp32 [N, T] tensor")
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    if n_tok_global is None:
        n_tok_global = max(int(mask.sum().item()), 1)
    o = out or _TbapFwd(N, T, dev)
    ws = workspace if workspace is not None else _workspace(dev, N, T)
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        args = (gen_logp.data_ptr(), ref_logp.data_ptr(), log_reward.data_ptr(), float(beta), int(K), _IS[is_mode],
                float(is_lo), float(is_hi), float(n_tok_global), ws.data_ptr(), o.seq_logp.data_ptr(),
                o.n_tokens.data_ptr(), o.adv.data_ptr(), o.coef.data_ptr(), o.partial.data_ptr())
        if grad_unscaled is None:
            check(L.tba_tbap_loss_fwd(ctypes.byref(x), *args, _ptr(st), _stream(dev)), "tba_tbap_loss_fwd")
        else:
            Nn, Tt, V = grad_unscaled.shape
            ors = grad_unscaled.stride(1) if Tt > 1 else (grad_unscaled.stride(0) if Nn > 1 else V)
            check(L.tba_tbap_loss_fwd_deferred(ctypes.byref(x), *args, grad_unscaled.data_ptr(),
                                               _DT[grad_unscaled.dtype], max(ors, V), _ptr(st), _stream(dev)),
                  "tba_tbap_loss_fwd_deferred")
    if st is not None:
        _raise_dev_status(st, "tba_tbap_loss_fwd")
    return o, ws


def lmhead_tbap_fwd(hidden, weight, tokens, mask, gen_logp, ref_logp, log_reward, beta: float, K: int,
                    is_mode: str = "clip", is_lo: float = 0.0, is_hi: float = 8.0, n_tok_global: float | None = None,
                    workspace=None, out: _TbapFwd | None = None, check_status: bool = _CHECK):
    """TBA' forward (Eq. 16) from hidden states (tba_lmhead_tbap_loss_fwd). Returns (_TbapFwd, workspace)."""
    L = _lib.load()
    x = make_lmhead(hidden, weight, tokens, mask)
    N, T = tokens.shape
    dev = hidden.device
    if gen_logp.shape != (N, T) or gen_logp.dtype != torch.float32 or not gen_logp.is_contiguous():
        raise ValueError("gen_logp must be a contiguous fp32 [N, T] tensor")
    for name, t in (("ref_logp", ref_logp), ("log_reward", log_reward)):
        if t.shape != (N,) or t.dtype != torch.float64 or t.device != dev or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous fp64 [N] tensor on {dev}")
    if n_tok_global is None:
        n_tok_global = max(int(mask.sum().item()), 1)
    o = out or _TbapFwd(N, T, dev)
    ws = workspace if workspace is not None else _lm_workspace(dev, N, T, weight.shape[0])
    st = _status(dev) if check_status else None
    with torch.cuda.device(dev):
        check(L.tba_lmhead_tbap_loss_fwd(ctypes.byref(x), gen_logp.data_ptr(), ref_logp.data_ptr(),
                                         log_reward.data_ptr(), float(beta), int(K), _IS[is_mode], float(is_lo),
                                         float(is_hi), float(n_tok_global), ws.data_ptr(), o.seq_logp.data_ptr(),
                                         o.n_tokens.data_ptr(), o.adv.data_ptr(), o.coef.data_ptr(),
                                         o.partial.data_ptr(), _ptr(st), _stream(dev)), "tba_lmhead_tbap_loss_fwd")
    if st is not None:
        _raise_dev_status(st, "tba_lmhead_tbap_loss_fwd")
    return o, ws


def tbap_bwd(logits, tokens, mask, workspace, coef, n_tok_global: float, grad_out=None, dlogits=None,
             dlogits_dtype=None):
    """Raw TBA' backward (tba_tbap_loss_bwd): dz = -(coef / n_tok_global) * g * (onehot - p)."""
    L = _lib.load()
    x = make_rows(logits, tokens, mask)
    dev = logits.device
    if dlogits is None:
        dlogits = torch.empty(logits.shape, dtype=dlogits_dtype or logits.dtype, device=dev)
    N, T, V = dlogits.shape
    ors = dlogits.stride(1) if T > 1 else (dlogits.stride(0) if N > 1 else V)
    if grad_out is not None:
        grad_out = grad_out.to(device=dev, dtype=torch.float64).contiguous()
    with torch.cuda.device(dev):
        check(L.tba_tbap_loss_bwd(ctypes.byref(x), workspace.data_ptr(), coef.data_ptr(), -1.0 / float(n_tok_global),
                                  _ptr(grad_out), dlogits.data_ptr(), _DT[dlogits.dtype], max(ors, V), _stream(dev)),
              "tba_tbap_loss_bwd")
    return dlogits


class TBAPrimeLoss(torch.autograd.Function):
    """Surrogate loss of the TBA' rule (Eq. 16); backward writes dlogits in one fused pass."""

    @staticmethod
    def forward(ctx, logits, tokens, mask, gen_logp, ref_logp, log_reward, beta, K, is_mode, is_lo, is_hi, n_tok,
                group, dlogits_dtype, aux):
        o, ws = tbap_fwd(logits, tokens, mask, gen_logp, ref_logp, log_reward, beta, K, is_mode, is_lo, is_hi, n_tok)
        if group is not None:
            import torch.distributed as dist
            dist.all_reduce(o.partial, op=dist.ReduceOp.SUM, group=group)
        ctx.save_for_backward(logits, tokens, mask, ws, o.coef)
        ctx.n_tok = n_tok
        ctx.dlogits_dtype = dlogits_dtype
        if aux is not None:
            aux.update(seq_logp=o.seq_logp, n_tokens=o.n_tokens, adv=o.adv, coef=o.coef, partial=o.partial)
        return o.partial[0]

    @staticmethod
    def backward(ctx, grad):
        logits, tokens, mask, ws, coef = ctx.saved_tensors
        d = tbap_bwd(logits, tokens, mask, ws, coef, ctx.n_tok, grad_out=grad, dlogits_dtype=ctx.dlogits_dtype)
        return (d,) + (None,) * 14


def tbap_loss(logits, tokens, mask, gen_logp, ref_logp, log_reward, beta: float, K: int, *, is_mode: str = "clip",
              is_lo: float = 0.0, is_hi: float = 8.0, n_tok_global=None, group=None, dlogits_dtype=None,
              return_aux: bool = False):
    """TBA' (Eq. 16) as an autograd-enabled surrogate loss. Defaults follow Table 5
    (CISPO IS bounds 0/8). n_tok_global (GRPO-style normaliser) defaults to the valid-token
    count of all ranks (one host sync + one all-reduce when `group` is given)."""
    if n_tok_global is None:
        n = mask.sum().to(torch.float64).reshape(1)
        if group is not None:
            import torch.distributed as dist
            dist.all_reduce(n, group=group)
        n_tok_global = max(float(n.item()), 1.0)
    aux = {} if return_aux else None
    loss = TBAPrimeLoss.apply(logits, tokens, mask, gen_logp, ref_logp, log_reward, float(beta), int(K), is_mode,
                              float(is_lo), float(is_hi), float(n_tok_global), group, dlogits_dtype, aux)
    return (loss, aux) if return_aux else loss


# ----------------------------------------------------------------------------- CUDA graphs
class CapturedStep:
    """Capture ``fn`` — a sequence of this library's calls on preallocated tensors (every call
    is stream-ordered, allocation-free in C and sync-free) — into a CUDA graph once, then
    ``replay()`` it. Removes the per-launch host overhead that dominates small shapes."""

    def __init__(self, fn, warmup: int = 2):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()

    def replay(self):
        self.graph.replay()
