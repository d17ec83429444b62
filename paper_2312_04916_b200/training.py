"""Early-exit training on B200: the fused exit-head loss and the weighted
multi-exit objective.

* `exit_head_loss_and_grads` / `ExitHeadCE` wrap `ee_exit_head_train`
  (include/ee.h): the tcgen05 fused head that computes an exit's weighted
  cross-entropy and its gradients without the (n, V) logits in HBM —
  replacing `run_head` + `cross_entropy` (eepipe/model.py:219-230,
  eepipe/autodiff.py:301-323).
* `TrainModel` / `weighted_loss` / `forward_all_exits` mirror
  `eepipe/model.py:233-285` with torch autograd for the backbone (the tape of
  the reference, `eepipe/autodiff.py:35-137`, is replaced by torch) and the
  fused head for every exit.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import ShapeError, TokenError
from .model import NORM_EPS, EarlyExitModel


def _torch():
    import torch
    return torch


_WS = {}


def _workspace(device, nbytes):
    torch = _torch()
    key = str(device)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def exit_head_loss_and_grads(x, W, targets, weight=1.0, dw_acc=None):
    """Fused exit head: returns (loss (0-d float32 tensor), dx (n, h) float32,
    dW (V, h) float32).  x (n, h) and W (V, h) bf16 CUDA tensors; targets
    int64 (n,).  dW is accumulated into ``dw_acc`` when given (microbatch
    accumulation, eepipe/pipeline.py:422-427)."""
    torch = _torch()
    _lib.require_cuda()
    if x.dim() != 2 or W.dim() != 2 or x.shape[1] != W.shape[1]:
        raise ShapeError(f"exit head: x {tuple(x.shape)} vs W {tuple(W.shape)}")
    n, h = x.shape
    V = W.shape[0]
    targets = targets.reshape(-1).to(device=x.device, dtype=torch.int64)
    if targets.numel() != n:
        raise ShapeError(f"{targets.numel()} targets for {n} rows")
    if n and (int(targets.min()) < 0 or int(targets.max()) >= V):
        raise TokenError("target id out of vocabulary range")
    x = x.to(torch.bfloat16).contiguous()
    W = W.to(torch.bfloat16).contiguous()
    lib = _lib.load()
    need = lib.ee_workspace_bytes(_lib.EE_OP_EXIT_HEAD_TRAIN, n, h, V, 0, 0)
    ws = _workspace(x.device, need)
    loss = torch.zeros((), dtype=torch.float32, device=x.device)
    dx = torch.empty((n, h), dtype=torch.float32, device=x.device)
    if dw_acc is None:
        dw_acc = torch.zeros((V, h), dtype=torch.float32, device=x.device)
    call("ee_exit_head_train", ptr(x), n, h, ptr(W), V, ptr(targets), float(weight),
         ptr(loss), ptr(dx), ptr(dw_acc), ptr(ws), ws.numel(), stream_ptr())
    return loss, dx, dw_acc


class ExitHeadCE:
    """torch.autograd.Function: weighted CE of one exit head.  The fused
    kernel produces loss and gradients in one call (the reference defers exit
    forwards into the backward step anyway, eepipe/pipeline.py:175-192), so
    backward only scales the saved gradients by the incoming grad."""

    _fn = None

    @classmethod
    def apply(cls, x, W, targets, weight=1.0):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, W, targets, weight):
                    loss, dx, dw = exit_head_loss_and_grads(x.detach(), W.detach(), targets,
                                                            weight)
                    ctx.save_for_backward(dx, dw)
                    ctx.dtypes = (x.dtype, W.dtype)
                    return loss

                @staticmethod
                def backward(ctx, g):
                    dx, dw = ctx.saved_tensors
                    return ((dx * g).to(ctx.dtypes[0]), (dw * g).to(ctx.dtypes[1]), None, None)

            cls._fn = _F
        return cls._fn.apply(x, W, targets, float(weight))
