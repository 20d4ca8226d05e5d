"""B200-native VarGrad trajectory-balance loss head (TBA, arXiv 2503.18929).

The compute lives in libtba.so (hand-written sm_100a CUDA, C ABI in include/tba.h);
this package only marshals PyTorch tensors into it. There is no CPU fallback: the ops
raise if the extension is missing.
"""
from ._lib import TbaError, load as load_library  # noqa: F401
from .dist import allreduce_partial_async, group_range, token_balanced_ranges  # noqa: F401
from .ops import (CapturedStep, LmHeadTBLoss, TBAPrimeLoss, VarGradTBLoss, lmhead_bwd_workspace_bytes,  # noqa: F401
                  lmhead_seq_logprob, lmhead_tb_loss, lmhead_tbap_bwd, lmhead_vargrad_bwd, lmhead_vargrad_fwd_bwd,
                  lmhead_fwd_bwd_workspace_bytes, lmhead_tbap_fwd, lmhead_token_logprob,
                  lmhead_vargrad_fwd,
                  lmhead_workspace_bytes, make_lmhead, make_rows, seq_logprob, tbap_bwd, tbap_fwd,  # noqa: F401
                  tbap_loss, token_logprob, vargrad_bwd, vargrad_fused, vargrad_fwd, vargrad_fwd_deferred, vargrad_pipelined,
                  vargrad_tb_loss,
                  vargrad_tb_loss_and_grad, workspace_bytes)

__all__ = ["CapturedStep", "seq_logprob", "token_logprob", "vargrad_tb_loss", "VarGradTBLoss", "vargrad_fwd", "vargrad_bwd", "workspace_bytes",
           "tbap_loss", "TBAPrimeLoss", "tbap_fwd", "tbap_bwd", "vargrad_fused", "vargrad_tb_loss_and_grad",
           "vargrad_fwd_deferred", "vargrad_pipelined", "lmhead_seq_logprob", "lmhead_vargrad_fwd", "lmhead_token_logprob",
           "lmhead_tbap_fwd", "lmhead_tb_loss", "LmHeadTBLoss", "lmhead_vargrad_bwd", "lmhead_tbap_bwd",
           "lmhead_bwd_workspace_bytes", "lmhead_vargrad_fwd_bwd", "lmhead_fwd_bwd_workspace_bytes",
           "lmhead_workspace_bytes", "make_lmhead",
           "group_range", "token_balanced_ranges", "allreduce_partial_async", "load_library", "TbaError"]
