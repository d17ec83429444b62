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
import os

import numpy as np

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import ShapeError, TokenError
from .model import NORM_EPS, EarlyExitModel


def _torch():
    import torch
    return torch


_WS = {}


def _workspace(device, nbytes, tag="head"):
    """Scratch buffer per (device, current stream, user): stage threads run on
    their own streams, so a buffer is never shared by concurrent kernels."""
    torch = _torch()
    key = (str(device), torch.cuda.current_stream(device).cuda_stream, tag)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


class _PinnedStaging:
    """Ring of reusable pinned host buffers for small host -> device uploads
    (token ids, targets): a slot is rewritten only after the copy that last
    read it has executed (its event).  Pinning a fresh tensor per upload
    (`Tensor.pin_memory`) costs ~1.6 ms of host time per call on this
    system, which made the training forward launch-bound."""

    def __init__(self, n=8):
        self.slots = [None] * n  # (pinned uint8 tensor, event)
        self.i = 0

    def upload(self, arr, device):
        torch = _torch()
        arr = np.ascontiguousarray(arr)
        nbytes = arr.nbytes
        i = self.i
        self.i = (i + 1) % len(self.slots)
        slot = self.slots[i]
        if slot is not None:
            slot[1].synchronize()  # the copy that last read this slot has run
        if slot is None or slot[0].numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8).pin_memory()
            slot = [buf, torch.cuda.Event()]
            self.slots[i] = slot
        host = slot[0][:nbytes]
        host.numpy()[:] = arr.reshape(-1).view(np.uint8)
        out = torch.empty(arr.shape, dtype=_TORCH_DTYPES[arr.dtype.str], device=device)
        out.view(-1).view(torch.uint8).copy_(host, non_blocking=True)
        slot[1].record(torch.cuda.current_stream(device))
        return out


_STAGING = {}
_TORCH_DTYPES = {}


def to_device_async(t, device):
    """Host tensor / array -> device without a stream synchronisation
    (pinned staging ring + non_blocking copy, per (device, stream))."""
    torch = _torch()
    if isinstance(t, torch.Tensor) and t.is_cuda:
        return t.to(device)
    a = t.numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    if not _TORCH_DTYPES:
        _TORCH_DTYPES.update({np.dtype(np.int64).str: torch.int64,
                              np.dtype(np.int32).str: torch.int32,
                              np.dtype(np.float32).str: torch.float32,
                              np.dtype(np.float64).str: torch.float64})
    dev = torch.device(device)
    if a.dtype.str not in _TORCH_DTYPES or a.size == 0:
        return torch.as_tensor(a).to(dev)
    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream)
    ring = _STAGING.get(key)
    if ring is None:
        ring = _STAGING[key] = _PinnedStaging()
    return ring.upload(a, dev)


def _check_ids(ids, V, what):
    """Range check on the HOST (a device-side check would synchronise)."""
    a = np.asarray(ids)
    if a.size and (int(a.min()) < 0 or int(a.max()) >= V):
        raise TokenError(f"{what} id out of vocabulary range")


def _head_inputs(x, W, targets, validated):
    """Shape / target checks and bf16 operands of the fused train head, plus
    its per-stream workspace."""
    torch = _torch()
    _lib.require_cuda()
    if x.dim() != 2 or W.dim() != 2 or x.shape[1] != W.shape[1]:
        raise ShapeError(f"exit head: x {tuple(x.shape)} vs W {tuple(W.shape)}")
    n, h = x.shape
    V = W.shape[0]
    if not isinstance(targets, torch.Tensor) or not targets.is_cuda:
        _check_ids(targets, V, "target")
        targets = to_device_async(np.asarray(targets, dtype=np.int64).reshape(-1), x.device)
    elif not validated and n and (int(targets.min()) < 0 or int(targets.max()) >= V):
        raise TokenError("target id out of vocabulary range")
    targets = targets.reshape(-1).to(dtype=torch.int64)
    if targets.numel() != n:
        raise ShapeError(f"{targets.numel()} targets for {n} rows")
    x = x.to(torch.bfloat16).contiguous()
    W = W.to(torch.bfloat16).contiguous()
    need = _lib.load().ee_workspace_bytes(_lib.EE_OP_EXIT_HEAD_TRAIN, n, h, V, 0, 0)
    return x, W, targets, _workspace(x.device, need)


def exit_head_loss_and_grads(x, W, targets, weight=1.0, dw_acc=None, validated=False):
    """Fused exit head: returns (loss (0-d float32 tensor), dx (n, h) float32,
    dW (V, h) float32).  x (n, h) and W (V, h) bf16 CUDA tensors; targets
    int64 (n,), host or device (``validated=True``: the caller has
    range-checked device targets on the host, so no synchronising check).
    dW is accumulated into ``dw_acc`` when given (microbatch accumulation,
    eepipe/pipeline.py:422-427)."""
    torch = _torch()
    x, W, targets, ws = _head_inputs(x, W, targets, validated)
    n, h = x.shape
    V = W.shape[0]
    loss = torch.zeros((), dtype=torch.float32, device=x.device)
    dx = torch.empty((n, h), dtype=torch.float32, device=x.device)
    if dw_acc is None:
        dw_acc = torch.zeros((V, h), dtype=torch.float32, device=x.device)
    call("ee_exit_head_train", ptr(x), n, h, ptr(W), V, ptr(targets), float(weight),
         ptr(loss), ptr(dx), ptr(dw_acc), ptr(ws), ws.numel(), stream_ptr())
    return loss, dx, dw_acc


class ExitHeadCE:
    """torch.autograd.Function: weighted CE of one exit head.  Without a
    float32 gradient sum on W the fused kernel produces loss and gradients in
    one call (the reference defers exit forwards into the backward step
    anyway, eepipe/pipeline.py:175-192) and backward scales them by the
    incoming gradient; with one (mixed precision) the head is split at the
    autograd boundary (ee_exit_head_train_fwd / _bwd) so the weight gradient
    lands in the sum inside the GEMM."""

    _fn = None

    @classmethod
    def apply(cls, x, W, targets, weight=1.0, validated=False):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, W, targets, weight, validated):
                    acc = getattr(W, "_ee_main_grad", None)
                    ctx.dtypes = (x.dtype, W.dtype)
                    ctx.split = acc is not None
                    if ctx.split:
                        # mixed precision: forward keeps d loss / d logits (G);
                        # the backward scales by the incoming gradient on the
                        # device and adds g * G^T x straight into W's float32
                        # sum inside the GEMM epilogue (no dW buffer, no pass)
                        x2, W2, t2, ws = _head_inputs(x.detach(), W.detach(), targets,
                                                      validated)
                        n, h = x2.shape
                        V = W2.shape[0]
                        G = torch.empty((n, V), dtype=torch.bfloat16, device=x2.device)
                        loss = torch.zeros((), dtype=torch.float32, device=x2.device)
                        call("ee_exit_head_train_fwd", ptr(x2), n, h, ptr(W2), V, ptr(t2),
                             float(weight), ptr(loss), ptr(G), ptr(ws), ws.numel(),
                             stream_ptr())
                        ctx.save_for_backward(x2, W2, G)
                        ctx.acc = acc
                        return loss
                    loss, dx, dw = exit_head_loss_and_grads(x.detach(), W.detach(), targets,
                                                            weight, validated=validated)
                    ctx.save_for_backward(dx, dw)
                    return loss

                @staticmethod
                def backward(ctx, g):
                    if ctx.split:
                        x2, W2, G = ctx.saved_tensors
                        n, h = x2.shape
                        V = W2.shape[0]
                        ws = _workspace(x2.device, _lib.load().ee_workspace_bytes(
                            _lib.EE_OP_EXIT_HEAD_TRAIN, n, h, V, 0, 0))
                        gs = g.detach().to(torch.float32).reshape(()).contiguous()
                        dx = torch.empty((n, h), dtype=torch.float32, device=x2.device)
                        call("ee_exit_head_train_bwd", ptr(x2), n, h, ptr(W2), V, ptr(G),
                             ptr(gs), ptr(dx), ptr(ctx.acc.view(V, h)), ptr(ws), ws.numel(),
                             stream_ptr())
                        return dx.to(ctx.dtypes[0]), None, None, None, None
                    dx, dw = ctx.saved_tensors
                    return (dx * g).to(ctx.dtypes[0]), (dw * g).to(ctx.dtypes[1]), None, None, None

            cls._fn = _F
        return cls._fn.apply(x, W, targets, float(weight), bool(validated))


# ---------------------------------------------------------------------------
# Trainable model: device parameters + forward pieces (eepipe/model.py)
# ---------------------------------------------------------------------------


class _ParamView(dict):
    """Compute parameters plus their float32 gradient accumulators (mixed
    mode): the backbone's linear layers send their weight gradients straight
    into ``main_grads`` (`ee_wgrad_accum`)."""

    def __init__(self, params, main_grads):
        super().__init__(params)
        self.main_grads = main_grads


_WGRAD_SIDE = {}
_WGRAD_OVERLAP = os.environ.get("EE_WGRAD_STREAM", "1") != "0"


def _wgrad_accum(x2, g2, acc):
    """acc (float32, in x out) += x2^T g2 (ee_wgrad_accum).  The weight
    gradient is off the backward's critical path (nothing downstream reads it
    before the optimizer), so it runs on a side stream of the current stream:
    its under-filled waves (64 tiles on 74 CTA pairs at 2048 x 2048) and
    tails overlap the input-gradient GEMMs.  `join_wgrad` orders the current
    stream after it (iteration end)."""
    torch = _torch()
    cur = torch.cuda.current_stream(x2.device)
    side = None
    if _WGRAD_OVERLAP:
        key = cur.cuda_stream
        side = _WGRAD_SIDE.get(key)
        if side is None:
            side = _WGRAD_SIDE[key] = torch.cuda.Stream(x2.device)
        side.wait_stream(cur)
    if side is None:
        call("ee_wgrad_accum", ptr(x2), ptr(g2), x2.shape[0], x2.shape[1], g2.shape[1], ptr(acc),
             stream_ptr())
        return
    call("ee_wgrad_accum", ptr(x2), ptr(g2), x2.shape[0], x2.shape[1], g2.shape[1], ptr(acc),
         ctypes.c_void_p(side.cuda_stream))
    x2.record_stream(side)
    g2.record_stream(side)


def _wgrad_accum_stacked(x2, g2, acc0, parts):
    """Weight gradients of `parts` adjacent matrices in one GEMM
    (ee_wgrad_accum_stacked): acc_j += x2^T g2[:, j N : (j + 1) N], g2 one
    (T, parts N) row-major matrix, acc_j = the float32 sums that follow acc0
    in the flat gradient buffer.  Same side stream as `_wgrad_accum`."""
    torch = _torch()
    T, K = x2.shape
    N = g2.shape[1] // parts
    cur = torch.cuda.current_stream(x2.device)
    side = None
    if _WGRAD_OVERLAP:
        key = cur.cuda_stream
        side = _WGRAD_SIDE.get(key)
        if side is None:
            side = _WGRAD_SIDE[key] = torch.cuda.Stream(x2.device)
        side.wait_stream(cur)
    st = ctypes.c_void_p(side.cuda_stream) if side is not None else stream_ptr()
    call("ee_wgrad_accum_stacked", ptr(x2), ptr(g2), T, K, N, parts, ptr(acc0), st)
    if side is not None:
        x2.record_stream(side)
        g2.record_stream(side)


def _adjacent(ts):
    """Equal-shape contiguous tensors stored back to back (the q / k / v
    weights, and their float32 sums, in the flat parameter buffers)."""
    t0 = ts[0]
    nb = t0.numel() * t0.element_size()
    return all(t.shape == t0.shape and t.dtype == t0.dtype and t.is_contiguous()
               and t.data_ptr() == t0.data_ptr() + i * nb for i, t in enumerate(ts))


def _row_ld(t):
    """Row stride of a (B, S, h) tensor whose rows are evenly spaced with
    unit column stride (a column block of a wider row-major buffer), else
    None."""
    if t.stride(-1) != 1 or (t.shape[0] > 1 and t.stride(0) != t.shape[1] * t.stride(1)):
        return None
    return t.stride(1)


def _column_blocks(gs):
    """The 2-D (T, N) views are consecutive column blocks of ONE row-major
    (T, len(gs) N) buffer (what the fused q / k / v projection and the
    attention backward produce): returns that buffer as a (T, len N) view,
    else None."""
    g0 = gs[0]
    T, N = g0.shape
    P = len(gs)
    for i, g in enumerate(gs):
        if (g.shape != g0.shape or g.dtype != g0.dtype or g.stride() != (P * N, 1)
                or g.data_ptr() != g0.data_ptr() + i * N * g0.element_size()):
            return None
    return g0.as_strided((T, P * N), (P * N, 1))


def join_wgrad(device=None):
    """Order the current stream after every weight-gradient accumulation
    issued from it (call before reading the float32 gradient sums)."""
    torch = _torch()
    cur = torch.cuda.current_stream(device)
    side = _WGRAD_SIDE.get(cur.cuda_stream)
    if side is not None:
        cur.wait_stream(side)


_OWN_LINEAR = os.environ.get("EE_LINEAR", "1") != "0"  # A/B switch: 0 = cuBLAS (torch)
# A/B switch: 0 = three q / k / v GEMMs each way instead of one stacked GEMM
_STACKED_QKV = os.environ.get("EE_STACKED_QKV", "1") != "0"
_STACKED_USES = [0]  # forward calls that took the stacked path (tests)


def _linear_fwd(x2, w, res2=None):
    """(T, N) bf16 = x2 (T, K) @ w (K, N) [+ res2] on the CTA-pair tcgen05
    GEMM (ee_linear_fwd; the residual is added before the one rounding)."""
    torch = _torch()
    T, K = x2.shape
    N = w.shape[1]
    if not _OWN_LINEAR:
        return x2 @ w if res2 is None else torch.addmm(res2, x2, w)
    out = torch.empty((T, N), dtype=x2.dtype, device=x2.device)
    call("ee_linear_fwd", ptr(x2), ptr(w), T, K, N, ptr(res2), ptr(out), stream_ptr())
    return out


def _linear_dgrad(g2, w, res2=None):
    """(T, K) bf16 = g2 (T, N) @ w (K, N)^T [+ res2] (ee_linear_dgrad; the
    addend is summed before the one rounding)."""
    torch = _torch()
    T, N = g2.shape
    K = w.shape[0]
    if not _OWN_LINEAR:
        return g2 @ w.t() if res2 is None else torch.addmm(res2, g2, w.t())
    out = torch.empty((T, K), dtype=g2.dtype, device=g2.device)
    call("ee_linear_dgrad", ptr(g2), ptr(w), T, K, N, ptr(res2) if res2 is not None else None,
         ptr(out), stream_ptr())
    return out


class _LinearFn:
    """y = x @ W (bf16) on the tcgen05 GEMM (ee_linear_fwd, residual folded
    in); the backward forms dX with ee_linear_dgrad and accumulates
    dW = X^T dY into the float32 main gradient (ee_wgrad_accum): no bf16
    weight gradient, returns None for W."""

    _fn = None

    @classmethod
    def get(cls):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, w, acc, res):
                    ctx.save_for_backward(x, w)
                    ctx.acc = acc
                    ctx.has_res = res is not None
                    x2 = x.reshape(-1, x.shape[-1]).contiguous()
                    # residual added by the GEMM itself (beta = 1): one rounding,
                    # no separate add pass over the (T, h) rows
                    r2 = res.reshape(-1, res.shape[-1]).contiguous() if res is not None else None
                    out = _linear_fwd(x2, w, r2)
                    return out.view(*x.shape[:-1], w.shape[1])

                @staticmethod
                def backward(ctx, gy):
                    x, w = ctx.saved_tensors
                    x2 = x.reshape(-1, x.shape[-1]).contiguous()
                    g2 = gy.reshape(-1, gy.shape[-1]).to(x2.dtype).contiguous()
                    gx = _linear_dgrad(g2, w).view(x.shape)
                    _wgrad_accum(x2, g2, ctx.acc)
                    return gx, None, None, (gy if ctx.has_res else None)

            cls._fn = _F
        return cls._fn


class _QKVFn:
    """q, k, v = h1 @ wq, h1 @ wk, h1 @ wv on the tcgen05 GEMM; the backward
    chains the three input-gradient GEMMs through the residual epilogue
    (dX = ((gq wq^T) + gk wk^T) + gv wv^T, one rounding per step, no
    separate add kernels) and accumulates the three weight gradients into
    their float32 sums (ee_wgrad_accum)."""

    _fn = None

    @classmethod
    def get(cls):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, wq, wk, wv, aq, ak, av):
                    x2 = x.reshape(-1, x.shape[-1]).contiguous()
                    ctx.save_for_backward(x2, wq, wk, wv)
                    ctx.acc = (aq, ak, av)
                    ctx.shape = x.shape
                    T, K = x2.shape
                    N = wq.shape[1]
                    ctx.stacked = (_STACKED_QKV and _adjacent((wq, wk, wv)) and _adjacent((aq, ak, av))
                                   and N % 128 == 0 and K % 128 == 0)
                    if ctx.stacked:
                        _STACKED_USES[0] += 1
                        # one GEMM over the adjacent weights; q, k, v are
                        # column blocks of one (T, 3N) buffer (the attention
                        # reads them in place through its row stride)
                        y = torch.empty((T, 3 * N), dtype=x2.dtype, device=x2.device)
                        call("ee_linear_fwd_stacked", ptr(x2), ptr(wq), T, K, N, 3, ptr(y),
                             stream_ptr())
                        y3 = y.view(*x.shape[:-1], 3 * N)
                        return y3[..., :N], y3[..., N:2 * N], y3[..., 2 * N:]
                    return tuple(_linear_fwd(x2, w).view(*x.shape[:-1], w.shape[1])
                                 for w in (wq, wk, wv))

                @staticmethod
                def backward(ctx, gq, gk, gv):
                    x2, wq, wk, wv = ctx.saved_tensors
                    if ctx.stacked and gq is not None and gk is not None and gv is not None:
                        gs = [g.reshape(-1, g.shape[-1]) for g in (gq, gk, gv)]
                        G = _column_blocks(gs) if gs[0].dtype == x2.dtype else None
                        if G is not None:
                            T, K = x2.shape
                            N = wq.shape[1]
                            gx = torch.empty((T, K), dtype=x2.dtype, device=x2.device)
                            call("ee_linear_dgrad_stacked", ptr(G), ptr(wq), T, K, N, 3, None,
                                 ptr(gx), stream_ptr())
                            _wgrad_accum_stacked(x2, G, ctx.acc[0], 3)
                            return gx.view(ctx.shape), None, None, None, None, None, None
                    gx = None
                    for g, w, acc in zip((gq, gk, gv), (wq, wk, wv), ctx.acc):
                        if g is None:
                            continue
                        g2 = g.reshape(-1, g.shape[-1]).to(x2.dtype).contiguous()
                        gx = _linear_dgrad(g2, w, gx)
                        _wgrad_accum(x2, g2, acc)
                    if gx is not None:
                        gx = gx.view(ctx.shape)
                    return gx, None, None, None, None, None, None

            cls._fn = _F
        return cls._fn


class _MLPFn:
    """GELU(x @ W1) @ W2 with the GELU fused into tcgen05 GEMM epilogues
    (csrc/mlp_train.cu): forward ee_mlp_up_gelu writes pre and act in one
    pass; backward ee_mlp_gelu_bwd forms dpre = (dY W2^T) * GELU'(pre) in the
    epilogue of the dgrad GEMM, and both weight gradients accumulate into the
    float32 sums with ee_wgrad_accum (eepipe/model.py:214-216)."""

    _fn = None

    @classmethod
    def get(cls):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, w1, w2, acc1, acc2, res):
                    x2 = x.reshape(-1, x.shape[-1]).contiguous()
                    T, h = x2.shape
                    N = w1.shape[1]
                    pre = torch.empty((T, N), dtype=x.dtype, device=x.device)
                    act = torch.empty((T, N), dtype=x.dtype, device=x.device)
                    call("ee_mlp_up_gelu", ptr(x2), ptr(w1), T, h, N, ptr(pre), ptr(act),
                         stream_ptr())
                    ctx.save_for_backward(x2, w1, w2, pre, act)
                    ctx.acc = (acc1, acc2)
                    ctx.shape = x.shape
                    ctx.has_res = res is not None
                    r2 = res.reshape(-1, res.shape[-1]).contiguous() if res is not None else None
                    return _linear_fwd(act, w2, r2).view(*x.shape[:-1], w2.shape[1])

                @staticmethod
                def backward(ctx, gy):
                    x2, w1, w2, pre, act = ctx.saved_tensors
                    acc1, acc2 = ctx.acc
                    T, h = x2.shape
                    N = w1.shape[1]
                    g2 = gy.reshape(-1, gy.shape[-1]).to(x2.dtype).contiguous()
                    dpre = torch.empty((T, N), dtype=x2.dtype, device=x2.device)
                    call("ee_mlp_gelu_bwd", ptr(g2), ptr(w2), T, h, N, ptr(pre), ptr(dpre),
                         stream_ptr())
                    _wgrad_accum(act, g2, acc2)
                    gx = _linear_dgrad(dpre, w1)
                    _wgrad_accum(x2, dpre, acc1)
                    return (gx.view(ctx.shape), None, None, None, None,
                            gy if ctx.has_res else None)

            cls._fn = _F
        return cls._fn


_MLP_FUSE = os.environ.get("EE_MLP_FUSE", "1") != "0"  # A/B switch (profiling)


def _mlp(params, prefix, h2, residual=None):
    """[residual +] GELU(h2 @ w1) @ w2 of a block; in mixed mode through the
    fused-GELU tcgen05 GEMMs (_MLPFn, residual added by the down GEMM), else
    plain torch."""
    torch = _torch()
    acc = getattr(params, "main_grads", None)
    n1, n2 = f"{prefix}.w1", f"{prefix}.w2"
    w1, w2 = params[n1], params[n2]
    if (_MLP_FUSE and acc is not None and n1 in acc and n2 in acc
            and h2.dtype == w1.dtype == torch.bfloat16
            and w1.shape[0] % 8 == 0 and w1.shape[1] % 8 == 0 and w2.shape[1] % 8 == 0
            and h2.is_cuda):
        return _MLPFn.get().apply(h2, w1, w2, acc[n1], acc[n2], residual)
    F = torch.nn.functional
    return _matmul(params, n2, F.gelu(_matmul(params, n1, h2)), residual)


def _matmul(params, name, x, residual=None):
    """[residual +] x @ params[name]; in mixed mode through the
    fused-accumulation linear (residual added by the GEMM)."""
    acc = getattr(params, "main_grads", None)
    w = params[name]
    if acc is not None and name in acc and x.dtype == w.dtype and w.shape[0] % 8 == 0 \
            and w.shape[1] % 8 == 0:
        return _LinearFn.get().apply(x, w, acc[name], residual)
    return x @ w if residual is None else residual + x @ w


def _flat_order(names):
    """Flat-buffer order of the parameters: as given, except that a block's
    q / k / v projections are placed back to back (wq, wk, wv) at the first
    of them, so the stacked GEMMs read them as one operand (stage partitions
    list their names sorted, which interleaves wo)."""
    have = set(names)
    out, done = [], set()
    for n in names:
        if n in done:
            continue
        prefix, _, leaf = n.rpartition(".")
        trio = [f"{prefix}.{w}" for w in ("wq", "wk", "wv")]
        if leaf in ("wq", "wk", "wv") and all(t in have for t in trio):
            out.extend(trio)
            done.update(trio)
        else:
            out.append(n)
            done.add(n)
    return out


class TrainModel:
    """Device-resident trainable copy of an `EarlyExitModel`: parameters as
    torch tensors (requires_grad) keyed by the reference names, compute dtype
    bf16 (the fused exit head runs on bf16 tensor cores).

    With ``master_dtype=torch.float32`` (mixed precision, what `train` uses)
    the bf16 leaves are views of one flat buffer and every microbatch's
    gradients are folded into float32 accumulators (one flat buffer) by one
    fused launch (`accumulate_grads`, ee_optimizer_step kind ACCUM); `grads()`
    then returns the float32 sums, and the optimizer writes the updated
    weights straight back into the bf16 leaves (`lp_params`)."""

    def __init__(self, model: EarlyExitModel, dtype=None, device=None, names=None,
                 master_dtype=None):
        torch = _torch()
        _lib.require_cuda()
        self.config = model.config
        self.heads = model.heads
        self.device = torch.device(device or "cuda:0")
        self.dtype = dtype or torch.bfloat16
        self.mixed = master_dtype is not None and master_dtype != self.dtype
        self.params = {}
        names = list(names if names is not None else model.params)
        srcs = {}
        for name in names:
            a = model.params[name].data
            srcs[name] = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
        if self.mixed:
            names = _flat_order(names)
            total = sum(srcs[n].numel() for n in names)
            self._flat = torch.empty(total, dtype=self.dtype, device=self.device)
            self._flat_grad = torch.zeros(total, dtype=torch.float32, device=self.device)
            self.main_grads = {}
            off = 0
            for name in names:
                t = srcs[name]
                k = t.numel()
                leaf = self._flat[off:off + k].view(t.shape)
                leaf.copy_(t.to(device=self.device))
                self.params[name] = leaf.requires_grad_()
                self.main_grads[name] = self._flat_grad[off:off + k].view(t.shape)
                leaf._ee_main_grad = self.main_grads[name]  # fused heads accumulate here
                off += k
        else:
            for name in names:
                self.params[name] = srcs[name].to(device=self.device,
                                                  dtype=self.dtype).detach().requires_grad_()

    def compute_params(self):
        if self.mixed:
            return _ParamView(self.params, self.main_grads)
        return self.params

    def zero_grad(self):
        for p in self.params.values():
            p.grad = None
        if self.mixed:
            self._flat_grad.zero_()

    def accumulate_grads(self):
        """Mixed precision: float32 accumulators += this microbatch's bf16
        gradients (one fused launch), then drop the bf16 gradients."""
        if not self.mixed:
            return
        torch = _torch()
        items = [(n, p) for n, p in self.params.items() if p.grad is not None]
        if not items:
            return
        table = np.zeros(len(items), dtype=_OPT_ENTRY)
        keep = []
        start = 0
        for i, (name, p) in enumerate(items):
            g = p.grad.to(self.dtype).contiguous()
            keep.append(g)
            acc = self.main_grads[name]
            table[i] = (acc.data_ptr(), g.data_ptr(), 0, 0, 0, acc.numel(), start)
            start += _pad4(acc.numel())
        tab = _device_table(table, self.device)
        call("ee_optimizer_step", ptr(tab), len(items), start, _lib.EE_OPT_ACCUM,
             _lib.dtype_code(self.dtype), 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, stream_ptr())
        for _, p in items:
            p.grad = None
        keep.append(tab)
        self._keep = keep  # alive until the next call (stream-ordered reuse)

    def grads(self):
        if self.mixed:
            join_wgrad(self.device)  # side-stream weight gradients (_wgrad_accum)
            return dict(self.main_grads)
        return {n: p.grad for n, p in self.params.items() if p.grad is not None}

    def lp_params(self):
        """bf16 leaves the optimizer may overwrite in place (mixed mode)."""
        return {n: p.detach() for n, p in self.params.items()} if self.mixed else {}


class _TableRing:
    """Asynchronous uploads of small host tables (numpy structured arrays)
    through a ring of pinned buffers: a buffer is refilled only after the
    copy that last read it has executed (its event), so no upload blocks the
    host on the stream (a pageable copy would synchronise every call)."""

    def __init__(self, n=4):
        self.slots = [None] * n  # (pinned uint8 tensor, device uint8 tensor, event)
        self.i = 0

    def upload(self, table, device):
        torch = _torch()
        raw = table.view(np.uint8)
        i = self.i
        self.i = (i + 1) % len(self.slots)
        slot = self.slots[i]
        if slot is None or slot[0].numel() < raw.size or slot[1].device != torch.device(device):
            cap = max(raw.size, 4096)
            slot = [torch.empty(cap, dtype=torch.uint8).pin_memory(),
                    torch.empty(cap, dtype=torch.uint8, device=device), None]
            self.slots[i] = slot
        if slot[2] is not None:
            slot[2].synchronize()
        slot[0].numpy()[:raw.size] = raw
        slot[1][:raw.size].copy_(slot[0][:raw.size], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(device))
        slot[2] = ev
        return slot[1]


_TABLES = {}


def _device_table(table, device):
    """Upload a small host table to the device without blocking the host
    (per-(device, stream) ring of pinned staging buffers)."""
    torch = _torch()
    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    ring = _TABLES.get(key)
    if ring is None:
        ring = _TABLES[key] = _TableRing()
    return ring.upload(table, device)


def _pad4(n):
    """Element offsets in a fused table start on 4-element boundaries so the
    kernel's 16-byte vector path applies to every aligned tensor."""
    return (n + 3) & ~3


class _RMSNormFn:
    """torch.autograd.Function over `ee_rmsnorm_fwd` / `ee_rmsnorm_bwd`
    (csrc/rmsnorm_train.cu): bf16 activations, float32 weight and
    statistics, deterministic weight gradient."""

    _fn = None

    @classmethod
    def get(cls):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, w, eps):
                    h = x.shape[-1]
                    x2 = x.reshape(-1, h).contiguous()
                    wf = w.detach().float().contiguous()
                    y = torch.empty_like(x2)
                    inv = torch.empty(x2.shape[0], dtype=torch.float32, device=x.device)
                    call("ee_rmsnorm_fwd", ptr(x2), x2.shape[0], h, ptr(wf), float(eps), ptr(y),
                         ptr(inv), stream_ptr())
                    ctx.save_for_backward(x2, wf, inv)
                    ctx.wdtype = w.dtype
                    return y.view(x.shape)

                @staticmethod
                def backward(ctx, gy):
                    x2, wf, inv = ctx.saved_tensors
                    n, h = x2.shape
                    gy2 = gy.reshape(n, h).to(torch.bfloat16).contiguous()
                    gx = torch.empty_like(x2)
                    gw = torch.empty(h, dtype=torch.float32, device=x2.device)
                    ws = _workspace(x2.device, _lib.load().ee_workspace_bytes(
                        _lib.EE_OP_RMSNORM_BWD, n, h, 0, 0, 0), tag="rmsnorm")
                    call("ee_rmsnorm_bwd", ptr(x2), ptr(wf), ptr(inv), ptr(gy2), None, n, h,
                         ptr(gx), ptr(gw), 0, ptr(ws), ws.numel(), stream_ptr())
                    return gx.view(gy.shape), gw.to(ctx.wdtype), None

            cls._fn = _F
        return cls._fn


class _NormForkFn:
    """(RMSNorm(x), x) of a pre-norm block: the second output is x itself for
    the block's residual branch, so the backward receives both gradients of x
    and `ee_rmsnorm_bwd` adds the residual one into gx in the same pass
    (no separate element-wise add over the (T, h) rows)."""

    _fn = None

    @classmethod
    def get(cls):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x, w, eps):
                    h = x.shape[-1]
                    x2 = x.reshape(-1, h).contiguous()
                    wf = w.detach().float().contiguous()
                    y = torch.empty_like(x2)
                    inv = torch.empty(x2.shape[0], dtype=torch.float32, device=x.device)
                    call("ee_rmsnorm_fwd", ptr(x2), x2.shape[0], h, ptr(wf), float(eps), ptr(y),
                         ptr(inv), stream_ptr())
                    ctx.save_for_backward(x2, wf, inv)
                    ctx.wdtype = w.dtype
                    return y.view(x.shape), x.view(x.shape)

                @staticmethod
                def backward(ctx, gy, gres):
                    x2, wf, inv = ctx.saved_tensors
                    n, h = x2.shape
                    gy2 = gy.reshape(n, h).to(torch.bfloat16).contiguous()
                    gr2 = (gres.reshape(n, h).to(torch.bfloat16).contiguous()
                           if gres is not None else None)
                    gx = torch.empty_like(x2)
                    gw = torch.empty(h, dtype=torch.float32, device=x2.device)
                    ws = _workspace(x2.device, _lib.load().ee_workspace_bytes(
                        _lib.EE_OP_RMSNORM_BWD, n, h, 0, 0, 0), tag="rmsnorm")
                    call("ee_rmsnorm_bwd", ptr(x2), ptr(wf), ptr(inv), ptr(gy2),
                         ptr(gr2) if gr2 is not None else None, n, h, ptr(gx), ptr(gw), 0,
                         ptr(ws), ws.numel(), stream_ptr())
                    return gx.view(gy.shape), gw.to(ctx.wdtype), None

            cls._fn = _F
        return cls._fn


def rmsnorm_fork(x, w, eps=NORM_EPS):
    """(rmsnorm(x, w), x) with both gradients of x joined inside the fused
    backward (bf16 on the GPU); elsewhere plain (rmsnorm(x, w), x)."""
    torch = _torch()
    if x.dtype == torch.bfloat16 and x.is_cuda and x.shape[-1] % 8 == 0:
        return _NormForkFn.get().apply(x, w, eps)
    return rmsnorm(x, w, eps), x


def rmsnorm(x, w, eps=NORM_EPS):
    """`eepipe/autodiff.py:228-244`.  bf16 activations go through the fused
    sm_100a kernels (`ee_rmsnorm_fwd/bwd`); float32 activations (the parity
    configuration of the tests) use float32 torch ops."""
    torch = _torch()
    if x.dtype == torch.bfloat16 and x.is_cuda and x.shape[-1] % 8 == 0:
        return _RMSNormFn.get().apply(x, w, eps)
    xf = x.float()
    inv = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (xf * inv * w.float()).to(x.dtype)


_SDPA = os.environ.get("EE_SDPA_BACKEND", "")  # profiling A/B: "", flash, efficient, cudnn


def _sdpa_backend():
    import contextlib
    if not _SDPA:
        return contextlib.nullcontext()
    from torch.nn.attention import SDPBackend, sdpa_kernel
    return sdpa_kernel({"flash": SDPBackend.FLASH_ATTENTION,
                        "efficient": SDPBackend.EFFICIENT_ATTENTION,
                        "cudnn": SDPBackend.CUDNN_ATTENTION}[_SDPA])


_OWN_ATTN = os.environ.get("EE_ATTN_TRAIN", "1") != "0"  # A/B switch: 0 = torch SDPA


class _AttnFn:
    """Causal attention of the training backbone on the tcgen05 kernels
    (ee_attn_train_fwd / _bwd, csrc/attention_train.cu): q, k, v (B, S, h)
    bf16 in the projections' own layout, output (B, S, h) straight into the
    wo GEMM (no (B, H, S, dh) transposes); lse saved for the backward
    (eepipe/autodiff.py:265-298)."""

    _fn = None

    @classmethod
    def get(cls):
        if cls._fn is None:
            torch = _torch()

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, q, k, v, num_heads):
                    B, S, h = q.shape
                    # q / k / v read in place when their rows are evenly
                    # spaced (column blocks of the fused projection's output)
                    q, k, v = (t if _row_ld(t) is not None else t.contiguous() for t in (q, k, v))
                    lq, lk, lv = (_row_ld(t) for t in (q, k, v))
                    o = torch.empty((B, S, h), dtype=q.dtype, device=q.device)
                    lse = torch.empty((B, num_heads, S), dtype=torch.float32, device=q.device)
                    call("ee_attn_train_fwd", ptr(q), lq, ptr(k), lk, ptr(v), lv, B, S, num_heads,
                         ptr(o), h, ptr(lse), stream_ptr())
                    ctx.save_for_backward(q, k, v, o, lse)
                    ctx.nh = num_heads
                    # gradients as column blocks of one (B, S, 3h) buffer when
                    # the inputs were (the fused q / k / v backward reads it)
                    ctx.packed = (lq == lk == lv == 3 * h and k.data_ptr() == q.data_ptr() + 2 * h
                                  and v.data_ptr() == q.data_ptr() + 4 * h)
                    return o

                @staticmethod
                def backward(ctx, do):
                    q, k, v, o, lse = ctx.saved_tensors
                    B, S, h = q.shape
                    do = do.to(q.dtype).contiguous()
                    if ctx.packed:
                        g = torch.empty((B, S, 3 * h), dtype=q.dtype, device=q.device)
                        dq, dk, dv = g[..., :h], g[..., h:2 * h], g[..., 2 * h:]
                        ld = 3 * h
                    else:
                        dq, dk, dv = (torch.empty((B, S, h), dtype=q.dtype, device=q.device)
                                      for _ in range(3))
                        ld = h
                    dsum = torch.empty_like(lse)
                    call("ee_attn_train_bwd", ptr(q), _row_ld(q), ptr(k), _row_ld(k), ptr(v),
                         _row_ld(v), ptr(o), h, ptr(do), h, ptr(lse), B, S, ctx.nh, ptr(dq), ld,
                         ptr(dk), ld, ptr(dv), ld, ptr(dsum), stream_ptr())
                    return dq, dk, dv, None

            cls._fn = _F
        return cls._fn


def causal_attention(q, k, v, num_heads):
    """(B, S, h) causal multi-head attention (`eepipe/autodiff.py:265-298`):
    the tcgen05 kernels for bf16, head_dim 128, S a multiple of 128 (every
    config's training shape); other shapes (the tests' tiny models) and
    float32 go through torch SDPA."""
    torch = _torch()
    B, S, h = q.shape
    dh = h // num_heads
    if (_OWN_ATTN and q.is_cuda and q.dtype == torch.bfloat16 and dh == 128 and S % 128 == 0):
        return _AttnFn.get().apply(q, k, v, num_heads)
    F = torch.nn.functional
    split = lambda t: t.view(B, S, num_heads, dh).transpose(1, 2)  # noqa: E731
    with _sdpa_backend():
        a = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
    return a.transpose(1, 2).reshape(B, S, h)


def _qkv(params, prefix, h1):
    """q, k, v projections; in mixed mode one autograd node (_QKVFn: chained
    input-gradient GEMMs, no add kernels)."""
    acc = getattr(params, "main_grads", None)
    names = [f"{prefix}.{w}" for w in ("wq", "wk", "wv")]
    ws = [params[n] for n in names]
    if (acc is not None and all(n in acc for n in names) and _OWN_LINEAR
            and all(w.dtype == h1.dtype and w.shape[0] % 8 == 0 and w.shape[1] % 8 == 0
                    for w in ws)):
        return _QKVFn.get().apply(h1, *ws, *(acc[n] for n in names))
    return tuple(_matmul(params, n, h1) for n in names)


def run_layer(params, prefix, x, num_heads):
    """One pre-norm block (`eepipe/model.py:207-216`).  The norms fork x so
    that the residual branch's gradient joins the norm's inside its backward
    kernel."""
    h1, x = rmsnorm_fork(x, params[f"{prefix}.attn_norm"])
    q, k, v = _qkv(params, prefix, h1)
    a = causal_attention(q, k, v, num_heads)
    x = _matmul(params, f"{prefix}.wo", a, residual=x)
    h2, x = rmsnorm_fork(x, params[f"{prefix}.mlp_norm"])
    return _mlp(params, prefix, h2, residual=x)


def head_input(params, head, x, num_heads):
    """Everything of `run_head` before the output projection
    (`eepipe/model.py:219-229`)."""
    torch = _torch()
    names = head.param_names
    if head.kind == "mlp+embed":
        h2 = rmsnorm(x, params[names["pre_norm"]])
        x = x + torch.nn.functional.gelu(h2 @ params[names["w1"]]) @ params[names["w2"]]
    elif head.kind == "layer+embed":
        x = run_layer(params, head.key, x, num_heads)
    if "norm" in names:
        x = rmsnorm(x, params[names["norm"]])
    return x


def run_head(params, head, x, num_heads):
    """Logits (B, S, V) of one head (`eepipe/model.py:219-230`) — the
    materialising API the reference exposes; training losses go through
    `head_loss` (fused, no logits)."""
    return head_input(params, head, x, num_heads) @ params[head.param_names["out"]].t()


def head_loss(params, head, x, targets, num_heads, validated=False):
    """Mean next-token CE of one head through the fused tcgen05 kernel
    (replaces run_head + cross_entropy, eepipe/model.py:219-230 +
    eepipe/autodiff.py:301-323).  ``validated``: device targets already
    range-checked on the host."""
    xi = head_input(params, head, x, num_heads)
    h = xi.shape[-1]
    W = params[head.param_names["out"]]
    return ExitHeadCE.apply(xi.reshape(-1, h), W, targets.reshape(-1), 1.0, validated)


def embed_tokens(params, tokens, max_seq_len):
    """`eepipe/model.py:233-243`."""
    torch = _torch()
    tokens = torch.as_tensor(np.asarray(tokens) if not isinstance(tokens, torch.Tensor) else tokens)
    if tokens.dim() != 2:
        raise ShapeError(f"tokens must be (batch, seq), got shape {tuple(tokens.shape)}")
    if tokens.shape[1] > max_seq_len:
        raise TokenError(f"sequence length {tokens.shape[1]} exceeds max_seq_len {max_seq_len}")
    V = params["tok_emb"].shape[0]
    if tokens.is_cuda:
        if tokens.numel() and (int(tokens.min()) < 0 or int(tokens.max()) >= V):
            raise TokenError("token id out of vocabulary range")
    else:
        _check_ids(tokens.numpy(), V, "token")
    dev = params["tok_emb"].device
    tokens = to_device_async(tokens, dev)
    pos = torch.arange(tokens.shape[1], device=dev)
    return params["tok_emb"][tokens] + params["pos_emb"][pos][None]


def forward_all_exits(model: TrainModel, tokens):
    """Logits at every head, depth order (`eepipe/model.py:246-261`)."""
    cfg = model.config
    wanted = {hd.layer_index for hd in model.heads}
    params = model.compute_params()
    x = embed_tokens(params, tokens, cfg.max_seq_len)
    taps = {0: x} if 0 in wanted else {}
    for i in range(1, cfg.num_layers + 1):
        x = run_layer(params, f"layer{i}", x, cfg.num_heads)
        if i in wanted:
            taps[i] = x
    return [run_head(params, hd, taps[hd.layer_index], cfg.num_heads) for hd in model.heads]


def weighted_loss(model: TrainModel, batch, weights):
    """Σ_i w_i · CE_i over heads in depth order; inputs batch[:, :-1],
    targets batch[:, 1:] (`eepipe/model.py:264-285`).  Returns (scalar
    tensor, per-exit float losses)."""
    torch = _torch()
    weights = list(weights)
    if len(weights) != len(model.heads):
        raise ShapeError(f"{len(weights)} weights for {len(model.heads)} exits (final included)")
    cfg = model.config
    batch = torch.as_tensor(np.asarray(batch) if not isinstance(batch, torch.Tensor) else batch)
    validated = not batch.is_cuda
    if validated:
        _check_ids(batch.numpy(), cfg.vocab_size, "token")
    batch = to_device_async(batch, model.device)
    wanted = {hd.layer_index for hd in model.heads}
    params = model.compute_params()
    x = embed_tokens(params, batch[:, :-1], cfg.max_seq_len)
    targets = batch[:, 1:]
    taps = {0: x} if 0 in wanted else {}
    for i in range(1, cfg.num_layers + 1):
        x = run_layer(params, f"layer{i}", x, cfg.num_heads)
        if i in wanted:
            taps[i] = x
    total = None
    per_exit = []
    for hd, w in zip(model.heads, weights):
        ce = head_loss(params, hd, taps[hd.layer_index], targets, cfg.num_heads, validated)
        per_exit.append(float(ce.detach()))
        term = ce * w
        total = term if total is None else total + term
    return total, per_exit


def single_device_gradients(model: TrainModel, batch, weights, microbatch_size):
    """Monolithic-model oracle of the pipeline: same microbatch split and
    accumulation order (`eepipe/pipeline.py:681-710`).  Returns (gradient
    map by name, per-exit mean losses)."""
    from .errors import ConfigError
    batch = np.asarray(batch)
    if batch.shape[0] % microbatch_size:
        raise ConfigError("batch does not divide into microbatches")
    num_mb = batch.shape[0] // microbatch_size
    model.zero_grad()
    sums = [0.0] * len(model.heads)
    for k in range(num_mb):
        loss, per_exit = weighted_loss(model, batch[k * microbatch_size:(k + 1) * microbatch_size],
                                       weights)
        loss.backward()
        model.accumulate_grads()  # mixed precision: fold into the float32 sums
        for i, v in enumerate(per_exit):
            sums[i] += v
    return model.grads(), {hd.key: sums[i] / num_mb for i, hd in enumerate(model.heads)}


# ---------------------------------------------------------------------------
# Optimizers and the training loop (eepipe/training.py)
# ---------------------------------------------------------------------------

_OPT_ENTRY = np.dtype([("param", "<u8"), ("grad", "<u8"), ("m", "<u8"), ("v", "<u8"),
                       ("param_lp", "<u8"), ("n", "<i8"), ("start", "<i8")])  # ee_opt_tensor_t


def _param_tensor(p):
    return getattr(p, "data", p)


class _FusedOptimizer:
    """Shared plumbing of `SGD` / `Adam`: one `ee_optimizer_step` launch over
    every parameter (include/ee.h, csrc/optim.cu).  Parameters are float32
    CUDA master tensors (``Param.data`` or bare tensors) updated in place;
    gradients float32 or bf16 of the same shapes."""

    kind = None

    def _launch(self, params, grads, scale, step_size, moments, lp=None):
        torch = _torch()
        names = sorted(grads)  # the reference's update order (eepipe/training.py:29, 46)
        if not names:
            return
        gdt = torch.float32 if any(grads[n].dtype != torch.bfloat16 for n in names) \
            else torch.bfloat16
        table = np.zeros(len(names), dtype=_OPT_ENTRY)
        keep = []
        start = 0
        dev = None
        for i, name in enumerate(names):
            p = _param_tensor(params[name])
            if not (isinstance(p, torch.Tensor) and p.is_cuda and p.dtype == torch.float32
                    and p.is_contiguous()):
                raise ShapeError(f"optimizer: {name} must be a contiguous float32 CUDA tensor")
            g = grads[name]
            if tuple(g.shape) != tuple(p.shape):
                raise ShapeError(f"optimizer: gradient of {name} has shape {tuple(g.shape)}, "
                                 f"parameter {tuple(p.shape)}")
            g = g.to(device=p.device, dtype=gdt).contiguous()
            dev = p.device
            keep.append(g)
            m, v = moments(name, p) if moments else (None, None)
            q = lp.get(name) if lp else None
            if q is not None and (q.dtype != torch.bfloat16 or q.numel() != p.numel()
                                  or not q.is_contiguous() or q.device != p.device):
                raise ShapeError(f"optimizer: low-precision copy of {name} must be a contiguous "
                                 "bf16 tensor of the same size on the same device")
            table[i] = (p.data_ptr(), g.data_ptr(), m.data_ptr() if m is not None else 0,
                        v.data_ptr() if v is not None else 0,
                        q.data_ptr() if q is not None else 0, p.numel(), start)
            start += _pad4(p.numel())
        tab = _device_table(table, dev)
        keep.append(tab)
        call("ee_optimizer_step", ptr(tab), len(names), start, self.kind, _lib.dtype_code(gdt),
             float(self.lr), float(getattr(self, "beta1", 0.0)), float(getattr(self, "beta2", 0.0)),
             float(getattr(self, "eps", 0.0)), float(scale), float(step_size), stream_ptr())
        return keep


class SGD(_FusedOptimizer):
    """p -= lr * scale * g (`eepipe/training.py:24-30`)."""

    kind = _lib.EE_OPT_SGD

    def __init__(self, lr):
        self.lr = lr

    def step(self, params, grads, scale, lp=None):
        self._launch(params, grads, scale, 0.0, None, lp)


class Adam(_FusedOptimizer):
    """Adam with the reference's update form (`eepipe/training.py:33-53`):
    m += (1-b1)(g-m); v += (1-b2)(g²-v);
    p -= lr·sqrt(1-b2^t)/(1-b1^t) · m/(sqrt(v)+eps); moments float32 on the
    parameter's device."""

    kind = _lib.EE_OPT_ADAM

    def __init__(self, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr = lr
        self.beta1 = beta1
        self.beta2 = beta2
        self.eps = eps
        self.m: dict = {}
        self.v: dict = {}
        self.t = 0

    def _moments(self, name, p):
        torch = _torch()
        if name not in self.m:
            self.m[name] = torch.zeros_like(p)
            self.v[name] = torch.zeros_like(p)
        return self.m[name], self.v[name]

    def step(self, params, grads, scale, lp=None):
        """``lp``: optional name -> bf16 tensor that receives the updated
        weights in the same launch (the compute copy of mixed precision)."""
        self.t += 1
        b1, b2 = self.beta1, self.beta2
        correction = np.sqrt(1 - b2 ** self.t) / (1 - b1 ** self.t)  # float64, as the reference
        self._launch(params, grads, scale, self.lr * correction, self._moments, lp)


def make_optimizer(kind, lr):
    from .errors import ConfigError
    if kind == "sgd":
        return SGD(lr)
    if kind == "adam":
        return Adam(lr)
    raise ConfigError(f"unknown optimizer {kind!r}")


def device_master(model: EarlyExitModel, device=None) -> EarlyExitModel:
    """float32 device copy of a model: the optimizer's master weights (the
    reference's monolithic float64 model, `eepipe/training.py:1-8`)."""
    torch = _torch()
    from .model import Param
    dev = torch.device(device or "cuda:0")
    params = {}
    for name, p in model.params.items():
        a = p.data
        t = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
        params[name] = Param(t.to(device=dev, dtype=torch.float32).contiguous().clone())
    return EarlyExitModel(model.config, params, model.heads)


def apply_update(optimizer, master, grads, computes, scale):
    """One fused optimizer launch over the float32 master weights; the
    updated weights are written straight into the first stage replica's bf16
    leaves, other replicas (tied embeddings on several stages) are copied."""
    lp, extra = {}, []
    for comp in computes:
        for name, t in comp.tm.lp_params().items():
            if name in lp or t.device != master.params[name].data.device:
                extra.append((t, name))
            else:
                lp[name] = t
    optimizer.step(master.params, grads, scale, lp=lp)
    for dst, name in extra:
        dst.copy_(master.params[name].data)


def train(run_cfg, corpus, metrics_path=None, progress=None, *, devices=None, dtype=None):
    """Train per the run configuration; returns (model, history)
    (`eepipe/training.py:64-136`).

    ``run_cfg`` carries the reference `RunConfig` fields this loop reads
    (model, seed, stages, microbatch_size, global_batch_size, steps,
    optimizer, learning_rate, data_seq_len, defer_exit_forward,
    fill_bubbles, weight_schedule()) — the reference's own RunConfig works
    as is; ``corpus.batch(rows, row_len, step)`` supplies token ids.  Every
    step partitions the float32 device master model, runs one 1F1B
    iteration (`pipeline.run_iteration_1f1b`: stage threads, fused tcgen05
    exit heads, bf16 compute, float32 gradient accumulation), and applies the fused optimizer with
    scale 1/num_microbatches.  Metrics: a header record then one record per
    step (losses, time, microbatches, weights) as line-delimited JSON.
    ``run_cfg.fill_bubbles``: every iteration also runs the
    plan_bubble_fill(stages, fill_f_over_b) fill microbatches, drawn from
    ``corpus.batch(n_fill * microbatch_size, row_len, step + 10**9)`` like the
    reference (`eepipe/training.py:76-101`)."""
    import json
    import time
    from .errors import ConfigError, NonFiniteError
    from .model import build_model, partition
    from .pipeline import IterationOptions, run_iteration_1f1b
    torch = _torch()
    _lib.require_cuda()
    master = device_master(build_model(run_cfg.model, run_cfg.seed),
                           devices[0] if devices else None)
    optimizer = make_optimizer(run_cfg.optimizer, run_cfg.learning_rate)
    rows_per_step = run_cfg.global_batch_size
    if rows_per_step % run_cfg.microbatch_size:
        raise ConfigError("global batch not divisible by the microbatch size")
    num_mb = rows_per_step // run_cfg.microbatch_size
    row_len = run_cfg.data_seq_len + 1
    schedule = run_cfg.weight_schedule() if hasattr(run_cfg, "weight_schedule") else None
    head_keys = None
    history = []
    fh = open(metrics_path, "w") if metrics_path else None

    def write(rec):
        if fh:
            fh.write(json.dumps(rec, sort_keys=True) + "\n")

    part = partition(master, run_cfg.stages, copy=False)
    plan, n_fill = None, 0
    if getattr(run_cfg, "fill_bubbles", False):
        from .bubblefill import plan_bubble_fill, truncated_part1_depths
        plan = plan_bubble_fill(run_cfg.stages, run_cfg.fill_f_over_b)
        depths = truncated_part1_depths(plan, part.exit_stages())
        n_fill = sum(1 for d in depths if d is not None) + plan.k_part2
    computes = []  # per-stage device state (bf16 weights, float32 gradient sums), kept
    try:
        for step in range(run_cfg.steps):
            batch = corpus.batch(rows_per_step, row_len, step)
            fill_batch = None
            if plan is not None and not plan.empty and n_fill:
                fill_batch = corpus.batch(n_fill * run_cfg.microbatch_size, row_len,
                                          step + 10**9)
            opts = IterationOptions(microbatch_size=run_cfg.microbatch_size,
                                    defer_exit_forward=getattr(run_cfg, "defer_exit_forward", True),
                                    weight_schedule=schedule, step=step, fill_plan=plan,
                                    fill_batch=fill_batch)
            t0 = time.perf_counter()
            grads, report = run_iteration_1f1b(part, batch, opts, model=master, devices=devices,
                                               dtype=dtype, master_dtype=torch.float32,
                                               stage_computes=computes)
            if not all(np.isfinite(v) for v in report.per_exit_losses.values()):
                raise NonFiniteError(f"non-finite loss at step {step}")
            apply_update(optimizer, master, grads, computes, 1.0 / num_mb)
            torch.cuda.synchronize()
            elapsed = time.perf_counter() - t0
            if head_keys is None:
                head_keys = [hd.key for hd in master.heads if hd.key in report.per_exit_losses]
                write({"record": "header", "heads": head_keys, "steps": run_cfg.steps,
                       "seed": run_cfg.seed})
            rec = {"record": "step", "step": step,
                   "losses": {k: report.per_exit_losses[k] for k in head_keys},
                   "time": elapsed, "microbatches": report.microbatches,
                   "weights": list(report.weights_used)}
            history.append(rec)
            write(rec)
            if progress is not None:
                progress(rec)
        if head_keys is None:
            write({"record": "header", "heads": [], "steps": 0, "seed": run_cfg.seed})
    finally:
        if fh:
            fh.close()
    return master, history


def trailing_average(values, window):
    """Mean of the last `window` entries at each step (`eepipe/training.py:144-150`)."""
    out = []
    for i in range(len(values)):
        lo = max(0, i - window + 1)
        out.append(float(np.mean(values[lo:i + 1])))
    return out
