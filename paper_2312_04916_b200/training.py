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


# ---------------------------------------------------------------------------
# Trainable model: device parameters + forward pieces (eepipe/model.py)
# ---------------------------------------------------------------------------


class TrainModel:
    """Device-resident trainable copy of an `EarlyExitModel`: parameters as
    torch tensors (requires_grad) keyed by the reference names, compute dtype
    bf16 (the fused exit head runs on bf16 tensor cores)."""

    def __init__(self, model: EarlyExitModel, dtype=None, device=None, names=None):
        torch = _torch()
        _lib.require_cuda()
        self.config = model.config
        self.heads = model.heads
        self.device = torch.device(device or "cuda:0")
        self.dtype = dtype or torch.bfloat16
        self.params = {}
        for name in (names if names is not None else model.params):
            a = model.params[name].data
            t = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
            self.params[name] = t.to(device=self.device, dtype=self.dtype).detach().requires_grad_()

    def zero_grad(self):
        for p in self.params.values():
            p.grad = None

    def grads(self):
        return {n: p.grad for n, p in self.params.items() if p.grad is not None}


def rmsnorm(x, w, eps=NORM_EPS):
    """`eepipe/autodiff.py:228-244` (float32 statistics)."""
    torch = _torch()
    xf = x.float()
    inv = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (xf * inv * w.float()).to(x.dtype)


def run_layer(params, prefix, x, num_heads):
    """One pre-norm block (`eepipe/model.py:207-216`)."""
    torch = _torch()
    F = torch.nn.functional
    B, S, h = x.shape
    dh = h // num_heads
    h1 = rmsnorm(x, params[f"{prefix}.attn_norm"])
    q, k, v = (h1 @ params[f"{prefix}.{w}"] for w in ("wq", "wk", "wv"))
    split = lambda t: t.view(B, S, num_heads, dh).transpose(1, 2)  # noqa: E731
    a = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
    x = x + a.transpose(1, 2).reshape(B, S, h) @ params[f"{prefix}.wo"]
    h2 = rmsnorm(x, params[f"{prefix}.mlp_norm"])
    return x + F.gelu(h2 @ params[f"{prefix}.w1"]) @ params[f"{prefix}.w2"]


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


def head_loss(params, head, x, targets, num_heads):
    """Mean next-token CE of one head through the fused tcgen05 kernel
    (replaces run_head + cross_entropy, eepipe/model.py:219-230 +
    eepipe/autodiff.py:301-323)."""
    xi = head_input(params, head, x, num_heads)
    h = xi.shape[-1]
    W = params[head.param_names["out"]]
    return ExitHeadCE.apply(xi.reshape(-1, h), W, targets.reshape(-1), 1.0)


def embed_tokens(params, tokens, max_seq_len):
    """`eepipe/model.py:233-243`."""
    torch = _torch()
    tokens = torch.as_tensor(np.asarray(tokens) if not isinstance(tokens, torch.Tensor) else tokens)
    if tokens.dim() != 2:
        raise ShapeError(f"tokens must be (batch, seq), got shape {tuple(tokens.shape)}")
    if tokens.shape[1] > max_seq_len:
        raise TokenError(f"sequence length {tokens.shape[1]} exceeds max_seq_len {max_seq_len}")
    V = params["tok_emb"].shape[0]
    if tokens.numel() and (int(tokens.min()) < 0 or int(tokens.max()) >= V):
        raise TokenError("token id out of vocabulary range")
    dev = params["tok_emb"].device
    tokens = tokens.to(dev)
    pos = torch.arange(tokens.shape[1], device=dev)
    return params["tok_emb"][tokens] + params["pos_emb"][pos][None]


def forward_all_exits(model: TrainModel, tokens):
    """Logits at every head, depth order (`eepipe/model.py:246-261`)."""
    cfg = model.config
    wanted = {hd.layer_index for hd in model.heads}
    x = embed_tokens(model.params, tokens, cfg.max_seq_len)
    taps = {0: x} if 0 in wanted else {}
    for i in range(1, cfg.num_layers + 1):
        x = run_layer(model.params, f"layer{i}", x, cfg.num_heads)
        if i in wanted:
            taps[i] = x
    return [run_head(model.params, hd, taps[hd.layer_index], cfg.num_heads) for hd in model.heads]


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
    batch = batch.to(model.device)
    wanted = {hd.layer_index for hd in model.heads}
    x = embed_tokens(model.params, batch[:, :-1], cfg.max_seq_len)
    targets = batch[:, 1:]
    taps = {0: x} if 0 in wanted else {}
    for i in range(1, cfg.num_layers + 1):
        x = run_layer(model.params, f"layer{i}", x, cfg.num_heads)
        if i in wanted:
            taps[i] = x
    total = None
    per_exit = []
    for hd, w in zip(model.heads, weights):
        ce = head_loss(model.params, hd, taps[hd.layer_index], targets, cfg.num_heads)
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
        for i, v in enumerate(per_exit):
            sums[i] += v
    return model.grads(), {hd.key: sums[i] / num_mb for i, hd in enumerate(model.heads)}
