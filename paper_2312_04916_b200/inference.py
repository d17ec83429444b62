"""Early-exit generation on B200: KV recomputation and pipeline-based inference.

Same API as the reference `eepipe.inference` (`eepipe/inference.py`):
`exit_decision`, `KVCache`, `DeferredToken`, `GenerationTrace`,
`generate_kv_recompute`, `generate_pipeline`, `greedy_reference`,
`compare_modes`, `default_stage_times`, `full_pass_units`.  The math runs in
libee.so (include/ee.h); this module is the host control logic: which rows
advance through which layers, where heads are evaluated, when a pass stops,
and the KV fill-mask discipline.

Design (B200-first):

* Weights are packed once per (model, dtype) into HBM in the layout the
  kernels stream: per layer Wqkv (3h, h), Wo (h, h), W1 (4h, h), W2 (h, 4h)
  K-major; head matrices stay (V, h).  KV cache is one (L, 2, s_max, h)
  tensor.  Residual rows are float32; weights/KV/GEMV inputs are float32
  (parity mode) or bf16 (perf mode).
* A pass keeps its rows in one device buffer ordered by entry depth
  DESCENDING, so the rows that advance at layer l (entry < l) are a suffix
  and the new token's row is simply appended — deferred hidden states never
  move between passes (the reference's `DeferredToken.hidden`).
* One C-ABI call advances a whole span of layers between head taps
  (`ee_decode_layers`); the host synchronises only at taps where the decide
  row's exit decision gates the rest of the pass (`run_pass` early stop,
  `eepipe/inference.py:324-326`).
* The fill mask of `KVCache` is kept on the host (positions are host-known
  control data) with the reference's refill / unfilled-read errors
  (`eepipe/inference.py:58-70`); the K/V values live only in HBM.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
from dataclasses import dataclass, field
from queue import Queue

import numpy as np

from . import _lib
from ._lib import EE_EPI_GELU, EE_EPI_RESIDUAL, call, ptr, stream_ptr
from .errors import ConfigError, NonFiniteError, TokenError
from .model import NORM_EPS, EarlyExitModel, HeadDesc, ModelConfig, StagePartition
from .schedule import inference_latency

_UNSUPPORTED_HEADS = ("layer+embed",)
_EMIT_TIMEOUT = 120.0
_HEAD_MAX_ROWS = 16
_MAPPED_RESULTS = os.environ.get("EE_MAPPED_RESULTS", "1") != "0"
_DEVICE_STAGE_STREAMS = {}
_RES_DTYPE = np.dtype([("tok", "<i4", (_HEAD_MAX_ROWS,)), ("conf", "<f4", (_HEAD_MAX_ROWS,)),
                       ("fire", "u1", (_HEAD_MAX_ROWS,)), ("bad", "<i4"), ("pad", "u1", (12,))])


def _torch():
    import torch
    return torch


def _device_stream(device):
    """The one CUDA stream every inference engine on a device runs on (kept
    for the process lifetime), keyed by the RESOLVED device index so 'cuda'
    and 'cuda:0' share it.  Engines allocate their buffers on it too, so the
    caching allocator never hands an engine's freed scratch to another
    stream while this one may still read it; pipeline stages placed on one
    GPU serialise their kernels in submission order (one GPU gains no
    throughput from overlapping its own stages)."""
    torch = _torch()
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    st = _DEVICE_STAGE_STREAMS.get(idx)
    if st is None:
        with torch.cuda.device(idx):
            st = _DEVICE_STAGE_STREAMS[idx] = torch.cuda.Stream(idx)
    return st


# ---------------------------------------------------------------------------
# Records (eepipe/inference.py:76-115)
# ---------------------------------------------------------------------------


@dataclass
class DeferredToken:
    """A generated token whose deep-layer KV entries are still missing.
    ``hidden`` is the device row index of its residual state (the state
    itself never leaves HBM)."""

    position: int
    exit_layer: int
    hidden: int


@dataclass
class GenerationTrace:
    prompt: list
    threshold: float
    mode: str
    tokens: list = field(default_factory=list)
    exit_layers: list = field(default_factory=list)
    exit_stages: list = field(default_factory=list)
    confidences: list = field(default_factory=list)  # per token: {head_key: float}
    latencies: list = field(default_factory=list)  # modeled, per token
    total_latency: float = 0.0
    baseline_latency: float = 0.0
    measured_latencies: list = field(default_factory=list)  # seconds, per token (host clock)
    measured_total: float = 0.0

    @property
    def speedup(self):
        return self.baseline_latency / self.total_latency if self.total_latency else 1.0

    @property
    def mean_exit_layer(self):
        return float(np.mean(self.exit_layers)) if self.exit_layers else 0.0

    def records(self):
        for i, tok in enumerate(self.tokens):
            yield {
                "position": len(self.prompt) + i,
                "token": int(tok),
                "exit_layer": self.exit_layers[i],
                "exit_stage": self.exit_stages[i] if self.exit_stages else None,
                "confidence": self.confidences[i],
                "latency": self.latencies[i] if i < len(self.latencies) else None,
                "measured_latency": (self.measured_latencies[i]
                                     if i < len(self.measured_latencies) else None),
            }


def exit_decision(logits, threshold):
    """Greedy decision at one exit (`eepipe/inference.py:118-133`):
    confidence = max softmax probability, token = argmax (lowest index wins),
    fire only on a strict crossing.  Evaluated on the GPU in float64; the
    generation paths use the fused kernel instead (`ee_exit_head_infer`)."""
    torch = _torch()
    _lib.require_cuda()
    z = torch.as_tensor(np.asarray(logits, dtype=np.float64).ravel()
                        if not isinstance(logits, torch.Tensor) else logits.reshape(-1))
    z = z.to(device="cuda", dtype=torch.float64)
    if not bool(torch.isfinite(z).all()):
        raise NonFiniteError("non-finite exit logits")
    if not 0.0 < threshold <= 1.0:
        raise ConfigError("threshold must lie in (0, 1]")
    p = torch.softmax(z, dim=0)
    token = int(torch.argmax(p))
    conf = float(p[token])
    return threshold < 1.0 and conf > threshold, token, conf


# ---------------------------------------------------------------------------
# KV cache (eepipe/inference.py:40-73)
# ---------------------------------------------------------------------------


class KVCache:
    """Per-layer key/value store in HBM with a monotone host-side fill mask.

    Layout: one (n_layers, 2, max_positions, num_heads*head_dim) tensor.
    `fill` raises ConfigError on a refill, `view` on a read below an unfilled
    position — the reference's KV-ordering guard."""

    def __init__(self, layer_indices, max_positions, num_heads, head_dim, dtype=None,
                 device=None):
        torch = _torch()
        self.layer_indices = list(layer_indices)
        self._slot = {l: i for i, l in enumerate(self.layer_indices)}
        self.max_positions = max_positions
        self.num_heads, self.head_dim = num_heads, head_dim
        self.data = torch.zeros((len(self.layer_indices), 2, max_positions, num_heads * head_dim),
                                dtype=dtype or torch.float32, device=device or "cuda")
        self.mask = np.zeros((len(self.layer_indices), max_positions), dtype=bool)

    def k(self, layer):
        return self.data[self._slot[layer], 0]

    def v(self, layer):
        return self.data[self._slot[layer], 1]

    def fill(self, layer, position, k, v):
        s = self._slot[layer]
        if self.mask[s, position]:
            raise ConfigError(f"KV at layer {layer}, position {position} already filled")
        self.data[s, 0, position] = _torch().as_tensor(np.asarray(k)).reshape(-1).to(self.data)
        self.data[s, 1, position] = _torch().as_tensor(np.asarray(v)).reshape(-1).to(self.data)
        self.mask[s, position] = True

    def view(self, layer, upto):
        s = self._slot[layer]
        if not self.mask[s, :upto].all():
            raise ConfigError(f"reading unfilled KV at layer {layer} below {upto}")
        shape = (upto, self.num_heads, self.head_dim)
        return self.data[s, 0, :upto].reshape(shape), self.data[s, 1, :upto].reshape(shape)

    def complete(self, upto):
        return bool(self.mask[:, :upto].all())

    def reset(self):
        self.mask[:] = False

    # bulk bookkeeping for kernel-side writes: layers [a, b) (slots), rows at
    # `positions` written, each row then reads [0, pos] (max_pos covers all)
    def mark_written(self, slot_a, slot_b, positions, max_pos):
        block = self.mask[slot_a:slot_b]
        if block[:, positions].any():
            bad = np.argwhere(block[:, positions])[0]
            raise ConfigError(f"KV at layer {self.layer_indices[slot_a + bad[0]]}, position "
                              f"{positions[bad[1]]} already filled")
        block[:, positions] = True
        if not block[:, :max_pos + 1].all():
            raise ConfigError(f"reading unfilled KV at layer {self.layer_indices[slot_a]} "
                              f"below {max_pos + 1}")


def _check_context(cfg: ModelConfig, needed):
    if needed > cfg.max_seq_len:
        raise TokenError(f"context of {needed} positions exceeds max_seq_len {cfg.max_seq_len}")


def default_stage_times(part: StagePartition):
    """`eepipe/inference.py:239-243`."""
    per = part.config.num_layers // part.num_stages
    return [per * 1.0 + 0.5 * len(st.heads) for st in part.stages]


def full_pass_units(cfg: ModelConfig, num_heads_total):
    """`eepipe/inference.py:246-248`."""
    return cfg.num_layers * 1.0 + 0.5 * num_heads_total


# ---------------------------------------------------------------------------
# Device engine: packed weights + KV + scratch for a layer span and heads
# ---------------------------------------------------------------------------


def _resolve_dtype(params, dtype):
    torch = _torch()
    if dtype is None:
        first = next(iter(params.values())).data
        if isinstance(first, np.ndarray):
            return torch.float32  # parity mode for reference-drawn weights
        return torch.float32 if first.dtype == torch.float32 else torch.bfloat16
    if isinstance(dtype, str):
        dtype = {"fp32": torch.float32, "float32": torch.float32, "bf16": torch.bfloat16,
                 "bfloat16": torch.bfloat16}[dtype]
    return dtype


class _Head:
    __slots__ = ("desc", "W", "norm", "pre_norm", "w1t", "w2t", "V")


class _PinnedRing:
    """Host->device staging of small int32 control arrays through a ring of
    pinned buffers; a buffer is rewritten only after the copy that last used
    it has executed (its event), so asynchronous uploads never race."""

    def __init__(self, cap, n=8):
        torch = _torch()
        self.cap = cap
        self.bufs = [torch.zeros(cap, dtype=torch.int32).pin_memory() for _ in range(n)]
        self.views = [b.numpy() for b in self.bufs]  # numpy views: no torch op per fill
        self.events = [None] * n
        self.i = 0

    def put(self, arr, dst, stream):
        torch = _torch()
        arr = np.asarray(arr, dtype=np.int32)
        n = arr.size
        if n > self.cap or n > dst.numel():
            raise ConfigError("control block overflow")
        i = self.i
        self.i = (i + 1) % len(self.bufs)
        if self.events[i] is not None:
            self.events[i].synchronize()
        self.views[i][:n] = arr
        # one raw cudaMemcpyAsync (no torch slicing / dispatch on the hot path)
        call("ee_copy_h2d", ctypes.c_void_p(dst.data_ptr()),
             ctypes.c_void_p(self.bufs[i].data_ptr()), 4 * n, ctypes.c_void_p(stream.cuda_stream))
        ev = self.events[i] or torch.cuda.Event()
        ev.record(stream)
        self.events[i] = ev


class Engine:
    """HBM-resident state of one inference worker (the whole model for KV
    recomputation, or one pipeline stage).  Built once per (params, dtype,
    device) and reused across generate calls."""

    def __init__(self, params, heads, cfg: ModelConfig, layer_indices, has_embedding, dtype,
                 device=None, max_rows=8):
        torch = _torch()
        _lib.require_cuda()
        self.device = torch.device(device or "cuda:0")
        self.cfg = cfg
        self.dtype = dtype
        self.dcode = _lib.dtype_code(dtype)
        self.layer_indices = list(layer_indices)
        self.h = h = cfg.hidden_dim
        self.nh = cfg.num_heads
        # construction runs on the device's engine stream, after whatever the
        # caller queued (device-initialised weights), and the caller's stream
        # waits for the packing before it may free or overwrite those weights
        caller = torch.cuda.current_stream(self.device)
        self.stream = _device_stream(self.device)
        self.stream.wait_stream(caller)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):

            def dev(name, dt=None):
                a = params[name].data
                t = torch.from_numpy(a) if isinstance(a, np.ndarray) else a
                return t.to(device=self.device, dtype=dt or dtype)

            self.tok_emb = dev("tok_emb").contiguous() if has_embedding else None
            self.pos_emb = dev("pos_emb").contiguous() if has_embedding else None
            self.kv = KVCache(self.layer_indices, cfg.max_seq_len, cfg.num_heads,
                              h // cfg.num_heads, dtype, self.device)
            # bf16 with h % 512 == 0: weights go to the tiled HBM layout of the
            # TMA-fed GEMV (one 16 KB bulk copy per pipeline stage)
            lib = _lib.load()
            self.tiled = (self.dcode == _lib.EE_BF16 and lib.ee_tiled_weight_bytes(h, h) > 0)
            self.wcode = _lib.EE_BF16_TILED if self.tiled else self.dcode

            def mat(t, col_scale=None):  # (N, K) row-major -> kernel layout
                t = t.contiguous()
                if not self.tiled:
                    return t
                out = torch.empty(lib.ee_tiled_weight_bytes(t.shape[0], t.shape[1]) // 2,
                                  dtype=torch.bfloat16, device=self.device)
                call("ee_pack_tiled", ptr(t), t.shape[0], t.shape[1], ptr(col_scale), ptr(out),
                     stream_ptr(self.stream))
                return out

            self.packed = []
            self.layers_c = (_lib.EeLayer * max(1, len(self.layer_indices)))()
            for i, l in enumerate(self.layer_indices):
                p = f"layer{l}."
                wqkv = torch.cat([dev(p + "wq").t(), dev(p + "wk").t(), dev(p + "wv").t()], 0)
                attn_norm = dev(p + "attn_norm", torch.float32).contiguous()
                mlp_norm = dev(p + "mlp_norm", torch.float32).contiguous()
                lw = {
                    # tiled mode folds the RMSNorm weights into the consuming
                    # matrices' columns (decode.cu)
                    "attn_norm": attn_norm,
                    "wqkv": mat(wqkv, attn_norm),
                    "wo": mat(dev(p + "wo").t()),
                    "mlp_norm": mlp_norm,
                    "w1": mat(dev(p + "w1").t(), mlp_norm),
                    "w2": mat(dev(p + "w2").t()),
                }
                del wqkv
                self.packed.append(lw)
                c = self.layers_c[i]
                for k in ("attn_norm", "wqkv", "wo", "mlp_norm", "w1", "w2"):
                    setattr(c, k, lw[k].data_ptr())
                c.kcache = self.kv.k(l).data_ptr()
                c.vcache = self.kv.v(l).data_ptr()
            self.heads = []
            for hd in heads:
                if hd.kind in _UNSUPPORTED_HEADS:
                    raise ConfigError(
                        f"head kind {hd.kind!r} is not supported for cached inference")
                e = _Head()
                e.desc = hd
                w_out = dev(hd.param_names["out"])
                e.V = w_out.shape[0]
                e.W = mat(w_out)
                del w_out
                e.norm = (dev(hd.param_names["norm"], torch.float32).contiguous()
                          if "norm" in hd.param_names else None)
                e.pre_norm = e.w1t = e.w2t = None
                if hd.kind == "mlp+embed":
                    e.pre_norm = dev(hd.param_names["pre_norm"], torch.float32).contiguous()
                    e.w1t = dev(hd.param_names["w1"]).t().contiguous()
                    e.w2t = dev(hd.param_names["w2"]).t().contiguous()
                self.heads.append(e)
            vmax = max([e.V for e in self.heads], default=1)
            self.head_ws = torch.zeros(
                _lib.load().ee_workspace_bytes(_lib.EE_OP_EXIT_HEAD, _HEAD_MAX_ROWS, h, vmax, 0, 0),
                dtype=torch.uint8, device=self.device)
            self.head_xn = torch.empty((_HEAD_MAX_ROWS, h), dtype=dtype, device=self.device)
            self.head_x = torch.empty((_HEAD_MAX_ROWS, h), dtype=torch.float32, device=self.device)
            self.head_mid = torch.empty((_HEAD_MAX_ROWS, 4 * h), dtype=dtype, device=self.device)
            self.max_slots = 256
            # per-evaluation result slots, packed so one D2H copy fetches them
            # all: tok int32[R] | conf f32[R] | fire u8[R] | bad int32 | pad
            self.res = torch.zeros(self.max_slots * _RES_DTYPE.itemsize, dtype=torch.uint8,
                                   device=self.device)
            self.h_res_t = torch.zeros(self.res.numel(), dtype=torch.uint8).pin_memory()
            self.h_res = self.h_res_t.numpy().view(_RES_DTYPE)
            self.h_tok, self.h_conf = self.h_res["tok"], self.h_res["conf"]
            self.h_fire, self.h_bad = self.h_res["fire"], self.h_res["bad"]
            self.max_rows = 0
            self._grow(max_rows)
        caller.wait_stream(self.stream)
        # accounting for bench.py: kernels launched and host<->device bytes
        self.launches = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    # -- scratch -------------------------------------------------------------
    def _grow(self, rows):
        torch = _torch()
        if rows <= self.max_rows:
            return
        rows = max(rows, 2 * self.max_rows)
        h, cfg = self.h, self.cfg
        self._x_old = getattr(self, "x", None)
        old_xb, old_ssq = getattr(self, "xb", None), getattr(self, "ssq", None)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self.x = torch.zeros((rows, h), dtype=torch.float32, device=self.device)
            # tiled mode: bf16 copy + sum-of-squares partials of the residual rows
            self.xb = torch.zeros((rows, h), dtype=torch.bfloat16, device=self.device)
            self.ssq = torch.zeros((rows, max(1, h // 16)), dtype=torch.float32,
                                   device=self.device)
            if old_xb is not None:
                self.xb[:old_xb.shape[0]].copy_(old_xb)
                self.ssq[:old_ssq.shape[0]].copy_(old_ssq)
            self.xn = torch.empty((rows, 4 * h), dtype=self.dtype, device=self.device)
            self.q = torch.empty((rows, h), dtype=torch.float32, device=self.device)
            self.attn = torch.empty((rows, h), dtype=self.dtype, device=self.device)
            wsb = _lib.load().ee_workspace_bytes(_lib.EE_OP_ATTENTION, rows, h, 0, cfg.num_heads,
                                                 cfg.max_seq_len)
            self.attn_ws = torch.zeros(wsb, dtype=torch.uint8, device=self.device)
            # control block: positions (rows) + gather lists, staged via pinned memory
            self.ctrl_cap = 4 * rows + 64 * _HEAD_MAX_ROWS + 64
            self.ctrl = torch.zeros(self.ctrl_cap, dtype=torch.int32, device=self.device)
            self.ring = _PinnedRing(self.ctrl_cap)
            self.ctrl_host = torch.zeros(2 * self.ctrl_cap, dtype=torch.int32).pin_memory()
            self.tokbuf = torch.zeros(2 * rows, dtype=torch.int32, device=self.device)
            if self.max_rows:
                old = self._x_old
                self.x[:old.shape[0]].copy_(old)
            # split-K partials of the multi-row (prefill) tcgen05 GEMM
            pfb = (_lib.load().ee_workspace_bytes(_lib.EE_OP_PREFILL, rows, h, 0, 0, 0)
                   if self.tiled and rows >= 17 else 0)
            self.pf_ws = torch.empty(max(pfb, 1), dtype=torch.uint8, device=self.device)
            self.pf_bytes = pfb  # handed to the decoder for prefill passes only
            self.dec = _lib.EeDecoder(h=h, nh=cfg.num_heads, s_max=cfg.max_seq_len,
                                      max_rows=rows, dtype=self.wcode, eps=NORM_EPS,
                                      x=self.x.data_ptr(), xb=self.xb.data_ptr(),
                                      ssq=self.ssq.data_ptr(),
                                      xn=self.xn.data_ptr(), q=self.q.data_ptr(),
                                      attn=self.attn.data_ptr(), ws=self.attn_ws.data_ptr(),
                                      ws_bytes=wsb,
                                      pf_ws=None, pf_ws_bytes=0)
        self.max_rows = rows
        self._x_old = None

    # -- primitives ------------------------------------------------------------
    def upload_ctrl(self, arr):
        self.ring.put(arr, self.ctrl, self.stream)
        self.h2d_bytes += 4 * len(arr)

    def ctrl_ptr(self, off):
        return ctypes.c_void_p(self.ctrl.data_ptr() + 4 * off)

    def embed_rows(self, tokens, positions, row0, out=None, staging=None, ctrl_off=None):
        """x[row0:row0+m] = tok_emb[tokens] + pos_emb[positions]  (or into
        ``out`` with a separate (ring, device buffer) ``staging`` pair, for an
        embedder running beside the stage worker that owns ``x``).  With
        ``ctrl_off`` the ids and positions were already uploaded with the
        pass's control block (ctrl[off:off+m], ctrl[off+m:off+2m])."""
        tokens = np.asarray(tokens, dtype=np.int64)
        if tokens.size and (tokens.min() < 0 or tokens.max() >= self.cfg.vocab_size):
            raise TokenError("token id out of vocabulary range")
        m = len(tokens)
        if out is None:
            self._grow(max(row0 + m, (m + 1) // 2))
            dst = ctypes.c_void_p(self.x.data_ptr() + 4 * row0 * self.h)
            ring, dbuf = self.ring, self.tokbuf
        else:
            dst = ptr(out)
            ring, dbuf = staging
        if ctrl_off is not None:
            tok_p, pos_p = self.ctrl_ptr(ctrl_off), self.ctrl_ptr(ctrl_off + m)
        else:
            stage = np.concatenate([tokens, np.asarray(positions, dtype=np.int64)])
            ring.put(stage, dbuf, _torch().cuda.current_stream(self.device))
            self.h2d_bytes += 4 * len(stage)
            tok_p, pos_p = ptr(dbuf), ctypes.c_void_p(dbuf.data_ptr() + 4 * m)
        stats = out is None and self.tiled and m > 0
        self.launches += 2 if stats else 1
        # embedding + (tiled mode) the new rows' statistics in one call
        call("ee_embed_stats", tok_p, pos_p, m, ptr(self.tok_emb), ptr(self.pos_emb), self.h,
             self.dcode, dst,
             ctypes.c_void_p(self.xb.data_ptr() + 2 * row0 * self.h) if stats else None,
             ctypes.c_void_p(self.ssq.data_ptr() + 4 * row0 * (self.h // 16)) if stats else None,
             stream_ptr(_torch().cuda.current_stream(self.device)))

    def refresh_stats(self, row0, m):
        """Tiled mode: bf16 copy + sum-of-squares partials of rows written
        outside the decoder (embedding, rows received from another stage)."""
        if not self.tiled or m == 0:
            return
        self.launches += 1
        call("ee_row_stats", ctypes.c_void_p(self.x.data_ptr() + 4 * row0 * self.h), self.h, m,
             self.h, ctypes.c_void_p(self.xb.data_ptr() + 2 * row0 * self.h),
             ctypes.c_void_p(self.ssq.data_ptr() + 4 * row0 * (self.h // 16)),
             stream_ptr(_torch().cuda.current_stream(self.device)))

    def eval_head(self, e: _Head, rows_ptr, m, threshold, slot, logits_dbg=None):
        """Fused head on m gathered rows of x; results into result slot."""
        h = self.h
        s = stream_ptr(self.stream)
        xsrc = self.x
        if e.desc.kind == "mlp+embed":
            # x' = x + GELU(RMSNorm(x; pre_norm) @ w1) @ w2   (eepipe/inference.py:178-182)
            call("ee_rmsnorm_rows", ptr(self.x), h, rows_ptr, m, h, None, NORM_EPS,
                 ptr(self.head_x), _lib.EE_F32, s)
            call("ee_rmsnorm_rows", ptr(self.head_x), h, None, m, h, ptr(e.pre_norm), NORM_EPS,
                 ptr(self.head_xn), self.dcode, s)
            call("ee_gemv", ptr(self.head_xn), m, h, ptr(e.w1t), 4 * h, self.dcode, EE_EPI_GELU,
                 ptr(self.head_mid), 4 * h, s)
            call("ee_gemv", ptr(self.head_mid), m, 4 * h, ptr(e.w2t), h, self.dcode,
                 EE_EPI_RESIDUAL, ptr(self.head_x), h, s)
            xsrc, rows_ptr = self.head_x, None
            self.launches += 4
        self.launches += 2  # row gather + norm, then the head GEMV
        call("ee_exit_head_infer", ptr(xsrc), h, rows_ptr, m, h, ptr(e.norm), NORM_EPS,
             ptr(e.W), e.V, self.wcode, float(threshold),
             self._res_ptr(slot, "tok"), self._res_ptr(slot, "conf"),
             self._res_ptr(slot, "fire"), self._res_ptr(slot, "bad"), ptr(logits_dbg),
             ptr(self.head_ws), self.head_ws.numel(), s)

    def native_engine(self):
        """The ee_engine_t view of this engine (rebuilt per call: scratch may
        have grown)."""
        lib_heads = getattr(self, "_heads_c", None)
        if lib_heads is None:
            kinds = {"minimalistic": 0, "norm+embed": 1, "mlp+embed": 2}
            arr = (_lib.EeHead * len(self.heads))()
            for i, e in enumerate(self.heads):
                hd = e.desc
                arr[i] = _lib.EeHead(hd.layer_index, int(hd.is_final), kinds[hd.kind],
                                     e.norm.data_ptr() if e.norm is not None else None,
                                     e.pre_norm.data_ptr() if e.pre_norm is not None else None,
                                     e.w1t.data_ptr() if e.w1t is not None else None,
                                     e.w2t.data_ptr() if e.w2t is not None else None,
                                     e.W.data_ptr(), e.V)
            self._heads_c = lib_heads = arr
        f = _RES_DTYPE.fields
        return _lib.EeEngine(
            ctypes.addressof(self.dec), ctypes.addressof(self.layers_c), len(self.layer_indices),
            ctypes.addressof(lib_heads), len(self.heads), self.dcode, self.wcode, NORM_EPS,
            self.tok_emb.data_ptr(), self.pos_emb.data_ptr(), self.ctrl.data_ptr(),
            self.ctrl_host.data_ptr(), self.ctrl_cap, self.head_ws.data_ptr(),
            self.head_ws.numel(), self.head_x.data_ptr(), self.head_xn.data_ptr(),
            self.head_mid.data_ptr(),
            # result slots: host-mapped pinned memory (the heads write them
            # directly; the loop polls each slot's last-written word instead
            # of a copy + stream synchronisation), or device memory + copy
            self.h_res_t.data_ptr() if _MAPPED_RESULTS else self.res.data_ptr(),
            self.h_res_t.data_ptr(),
            _RES_DTYPE.itemsize, self.max_slots, f["tok"][1], f["conf"][1], f["fire"][1],
            f["bad"][1], self.stream.cuda_stream,
            self.pf_ws.data_ptr() if self.pf_bytes else None, self.pf_bytes)

    def _res_ptr(self, slot, field):
        return ctypes.c_void_p(self.res.data_ptr() + slot * _RES_DTYPE.itemsize +
                               _RES_DTYPE.fields[field][1])

    def fetch_results(self, nslots):
        """One D2H copy of the first nslots result slots, then synchronise;
        results are read through the numpy views h_tok / h_conf / h_fire."""
        if nslots == 0:
            return
        nb = nslots * _RES_DTYPE.itemsize
        self.h_res_t[:nb].copy_(self.res[:nb], non_blocking=True)
        self.d2h_bytes += nb
        self.stream.synchronize()
        if self.h_bad[:nslots].any():
            raise NonFiniteError("non-finite exit logits")

    def run_layers(self, la, lb, n_rows, m_active, max_pos, pos_off, prefill=False):
        """Slots [la, lb) of this engine's layers over rows [0, n_rows).
        ``prefill``: the pass carries the prompt rows (computed once in every
        mode) and may use the multi-row tcgen05 GEMM; decode passes always
        take the row-stable GEMV."""
        n = lb - la
        if n <= 0:
            return
        arr = (ctypes.c_int32 * n)(*m_active)
        layers = ctypes.c_void_p(ctypes.addressof(self.layers_c) +
                                 la * ctypes.sizeof(_lib.EeLayer))
        def per(v):  # kernels per layer (decode.cu decode_layer_launches)
            if not self.tiled:
                return 7
            return 9 if prefill and self.pf_bytes and v >= 17 else 5
        self.launches += sum(per(v) for v in m_active if v)
        if prefill and self.pf_bytes:
            self.dec.pf_ws, self.dec.pf_ws_bytes = self.pf_ws.data_ptr(), self.pf_bytes
        try:
            call("ee_decode_layers", ctypes.byref(self.dec), layers, n, n_rows, arr,
                 self.ctrl_ptr(pos_off), int(max_pos), stream_ptr(self.stream))
        finally:
            self.dec.pf_ws, self.dec.pf_ws_bytes = None, 0


_ENGINE_CACHE_ATTR = "_ee_engines"


def _engine_for(owner, params, heads, cfg, layer_indices, has_embedding, dtype, device=None):
    """Engines are cached on the owning object (model or stage spec)."""
    torch = _torch()
    dt = _resolve_dtype(params, dtype)
    dev = torch.device(device or "cuda:0")
    cache = owner.__dict__.setdefault(_ENGINE_CACHE_ATTR, {})
    key = (dt, str(dev), tuple(layer_indices), tuple(hd.key for hd in heads))
    eng = cache.get(key)
    if eng is None:
        eng = Engine(params, heads, cfg, layer_indices, has_embedding, dt, dev)
        cache[key] = eng
    return eng


# ---------------------------------------------------------------------------
# KV recomputation (single worker) — eepipe/inference.py:256-381
# ---------------------------------------------------------------------------


def generate_kv_recompute(model: EarlyExitModel, prompt, threshold, max_new_tokens,
                          max_deferred=4, *, dtype=None, device=None) -> GenerationTrace:
    """Incremental decoding that batches deferred early-exit tokens into the
    current pass to recompute their missing KV entries
    (`eepipe/inference.py:256-381`).  ``dtype`` selects fp32 parity mode or
    bf16 perf mode (default: fp32 for host float64 weights, else the weights'
    dtype)."""
    if max_deferred < 1:
        raise ConfigError("max_deferred must be at least 1")
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise ConfigError("prompt must be non-empty")
    if not 0.0 < threshold <= 1.0:
        raise ConfigError("threshold must lie in (0, 1]")
    cfg = model.config
    _check_context(cfg, len(prompt) + max_new_tokens)
    L = cfg.num_layers
    eng = _engine_for(model, model.params, model.heads, cfg, range(1, L + 1), True, dtype, device)
    torch = _torch()
    with torch.cuda.device(eng.device), torch.cuda.stream(eng.stream):
        return _kv_recompute(eng, model, prompt, threshold, max_new_tokens, max_deferred)


def _kv_recompute(eng, model, prompt, threshold, max_new_tokens, max_deferred):
    """One native call runs the whole decode loop (`ee_generate_kv_recompute`,
    csrc/recompute.cu: prefill, per-token batched back-fill passes with the
    exit decisions, flush, KV completeness); this wrapper validates, sizes
    the scratch and turns the outputs into a `GenerationTrace`."""
    cfg = model.config
    L = cfg.num_layers
    tok = np.asarray(prompt, dtype=np.int64)
    if tok.min() < 0 or tok.max() >= cfg.vocab_size:
        raise TokenError("token id out of vocabulary range")
    t0 = len(prompt)
    eng.kv.reset()
    eng._grow(max(t0, max_deferred + 1))
    n_heads = len(eng.heads)
    prompt32 = np.ascontiguousarray(tok, dtype=np.int32)
    out_tok = np.zeros(max_new_tokens, dtype=np.int32)
    out_exit = np.zeros(max_new_tokens, dtype=np.int32)
    out_depth = np.zeros(max_new_tokens, dtype=np.int32)
    out_lat = np.zeros(max_new_tokens, dtype=np.float64)
    conf = np.full((cfg.max_seq_len, n_heads), np.nan, dtype=np.float32)
    kv_mask = np.zeros((L, cfg.max_seq_len), dtype=np.uint8)
    engine = eng.native_engine()
    args = _lib.EeGenerateArgs(
        ctypes.addressof(engine), prompt32.ctypes.data, t0, max_new_tokens, max_deferred,
        cfg.max_seq_len, _HEAD_MAX_ROWS, float(threshold), n_heads, out_tok.ctypes.data,
        out_exit.ctypes.data, out_depth.ctypes.data, out_lat.ctypes.data, conf.ctypes.data,
        kv_mask.ctypes.data, 0, 0, 0.0, 0, 0, 0)
    call("ee_generate_kv_recompute", ctypes.byref(args))
    eng.launches += args.launches
    eng.h2d_bytes += args.h2d_bytes + 4 * t0
    eng.d2h_bytes += args.d2h_bytes
    eng.kv.mask[:] = kv_mask.astype(bool)
    gen = args.n_generated
    units = full_pass_units(cfg, len(model.heads))
    trace = GenerationTrace(prompt, threshold, "recompute")
    trace.tokens = [int(t) for t in out_tok[:gen]]
    trace.exit_layers = [int(e) for e in out_exit[:gen]]
    trace.measured_latencies = [float(v) for v in out_lat[:gen]]
    trace.measured_total = float(args.total_s)
    keys = [e.desc.key for e in eng.heads]
    trace.confidences = []
    for i in range(gen):
        row = conf[t0 - 1 + i]
        trace.confidences.append({keys[k]: float(row[k]) for k in range(n_heads)
                                  if not np.isnan(row[k])})
    trace.latencies = [units * int(d) / L for d in out_depth[:gen]]
    trace.total_latency = sum(trace.latencies) + (units if args.flushed else 0.0)
    trace.baseline_latency = units * gen
    return trace


# ---------------------------------------------------------------------------
# Pipeline mode — eepipe/inference.py:389-539
# ---------------------------------------------------------------------------


@dataclass
class _FwdMsg:
    rows: object  # device tensor (m, h) float32
    positions: list
    decide_pos: int
    emitted: bool
    ready: object = None  # CUDA event recorded on the sender's stream
    stop: bool = False


@dataclass
class _EmitMsg:
    position: int
    token: int
    exit_layer: int
    exit_stage: int


class _InferStage:
    """One pipeline stage: own layers, heads, KV cache and CUDA stream;
    strict FIFO position order (`eepipe/inference.py:406-463`)."""

    def __init__(self, spec, cfg, threshold, q_in, q_out, emit_q, conf_log, lock, dtype, device):
        torch = _torch()
        heads = [hd for _, hd in spec.heads]
        self.spec = spec
        self.cfg = cfg
        self.threshold = threshold
        self.eng = _engine_for(spec, spec.params, heads, cfg, spec.layer_indices,
                               spec.has_embedding, dtype, device)
        self.eng.kv.reset()
        # every engine on a device runs on that device's one stream
        # (_device_stream): stages on one GPU serialise in submission order
        self.stream = self.eng.stream
        self.heads_at = {}
        for local, hd in spec.heads:
            hi = next(i for i, e in enumerate(self.eng.heads) if e.desc.key == hd.key)
            self.heads_at.setdefault(local, []).append(hi)
        self.q_in, self.q_out, self.emit_q = q_in, q_out, emit_q
        self.conf_log, self.lock = conf_log, lock
        self.exception = None

    def _check_heads(self, msg, local, n):
        e = self.eng
        if local not in self.heads_at or msg.decide_pos not in msg.positions:
            return
        r = msg.positions.index(msg.decide_pos)
        e.upload_ctrl(list(msg.positions) + [r])
        for k, hi in enumerate(self.heads_at[local]):
            e.eval_head(e.heads[hi], e.ctrl_ptr(n), 1, self.threshold, k)
        e.fetch_results(len(self.heads_at[local]))
        for k, hi in enumerate(self.heads_at[local]):
            hd = e.heads[hi].desc
            conf = float(e.h_conf[k, 0])
            with self.lock:
                self.conf_log.setdefault(msg.decide_pos, {})[hd.key] = conf
            if not msg.emitted and (bool(e.h_fire[k, 0]) or hd.is_final):
                self.emit_q.put(_EmitMsg(msg.decide_pos, int(e.h_tok[k, 0]), hd.layer_index,
                                         self.spec.index))
                msg.emitted = True

    def run(self):
        torch = _torch()
        try:
            with torch.cuda.device(self.eng.device), torch.cuda.stream(self.stream):
                e = self.eng
                while True:
                    msg = self.q_in.get()
                    if msg.stop:
                        if self.q_out is not None:
                            self.q_out.put(msg)
                        return
                    if msg.ready is not None:
                        self.stream.wait_event(msg.ready)
                    n = len(msg.positions)
                    e._grow(n)
                    e.x[:n].copy_(msg.rows, non_blocking=True)
                    msg.rows.record_stream(self.stream)
                    e.refresh_stats(0, n)
                    e.upload_ctrl(list(msg.positions))
                    self._check_heads(msg, 0, n)
                    max_pos = max(msg.positions)
                    local = 1
                    stops = sorted(k for k in self.heads_at if k >= 1)
                    nloc = len(self.spec.layer_indices)
                    if not stops or stops[-1] != nloc:
                        stops.append(nloc)
                    for stop in stops:
                        if stop >= local:
                            e.upload_ctrl(list(msg.positions))
                            # the prompt message (positions 0..t0-1) is the prefill
                            e.run_layers(local - 1, stop, n, [n] * (stop - local + 1), max_pos, 0,
                                         prefill=msg.positions[0] == 0)
                            e.kv.mark_written(local - 1, stop, list(msg.positions), max_pos)
                            self._check_heads(msg, stop, n)
                            local = stop + 1
                    if self.q_out is not None:
                        out = e.x[:n].clone()
                        ev = torch.cuda.Event()
                        ev.record(self.stream)
                        self.q_out.put(_FwdMsg(out, msg.positions, msg.decide_pos, msg.emitted,
                                               ev))
        except BaseException as exc:  # surfaced by the coordinator
            self.exception = exc
            self.emit_q.put(exc)


def generate_pipeline(part: StagePartition, prompt, threshold, max_new_tokens, stage_times=None,
                      *, dtype=None, devices=None) -> GenerationTrace:
    """Pipeline-based early-exit inference (`eepipe/inference.py:466-539`).

    One worker thread per stage, each with its own CUDA stream (and its own
    GPU when ``devices`` lists several): stage s processes positions strictly
    in order; the emitted token's pass continues to the last stage filling KV
    while stage 1 already runs the next token.  For the multi-process
    NCCL/NVLink variant (one process per GPU) see `pipeline_infer.py`."""
    torch = _torch()
    if part.num_stages < 2:
        raise ConfigError("pipeline inference needs at least 2 stages")
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise ConfigError("prompt must be non-empty")
    if not 0.0 < threshold <= 1.0:
        raise ConfigError("threshold must lie in (0, 1]")
    cfg = part.config
    _check_context(cfg, len(prompt) + max_new_tokens)
    _lib.require_cuda()
    if devices is None:
        devices = ["cuda:0"] * part.num_stages
    conf_log: dict = {}
    lock = threading.Lock()
    queues = [Queue() for _ in range(part.num_stages)]
    emit_q: Queue = Queue()
    stages = []
    for i, spec in enumerate(part.stages):
        q_out = queues[i + 1] if i + 1 < part.num_stages else None
        stages.append(_InferStage(spec, cfg, threshold, queues[i], q_out, emit_q, conf_log, lock,
                                  dtype, devices[i % len(devices)]))
    threads = [threading.Thread(target=s.run, daemon=True, name=f"infer-stage-{s.spec.index}")
               for s in stages]
    # the stage workers and the coordinator are latency-bound Python threads
    # that mostly wait in CUDA / queue calls: hand the GIL over quickly
    import sys
    old_switch = sys.getswitchinterval()
    sys.setswitchinterval(5e-5)
    for t in threads:
        t.start()

    first = stages[0].eng
    t0 = len(prompt)
    trace = GenerationTrace(prompt, threshold, "pipeline")
    # the coordinator embeds on its own stream with its own staging buffers
    # (stage 1's worker owns first.x and first.ring)
    with torch.cuda.device(first.device):
        emb_stream = getattr(first, "_emb_stream", None)
        if emb_stream is None:
            emb_stream = first._emb_stream = torch.cuda.Stream(first.device)
        emb_stream.wait_stream(first.stream)  # embedding tables packed on the engine stream
        cap = 2 * max(t0, 1) + 16
        with torch.cuda.stream(emb_stream):
            staging = (_PinnedRing(cap), torch.zeros(cap, dtype=torch.int32, device=first.device))

    def embedded(tokens, positions):
        with torch.cuda.device(first.device), torch.cuda.stream(emb_stream):
            rows = torch.empty((len(tokens), cfg.hidden_dim), dtype=torch.float32,
                               device=first.device)
            first.embed_rows(tokens, positions, 0, out=rows, staging=staging)
            ev = torch.cuda.Event()
            ev.record(emb_stream)
        return rows, ev

    t_start = time.perf_counter()
    t_last = t_start
    rows, ev = embedded(prompt, list(range(t0)))
    queues[0].put(_FwdMsg(rows, list(range(t0)), t0 - 1, False, ev))
    position = t0 - 1
    try:
        for i in range(max_new_tokens):
            emit = emit_q.get(timeout=_EMIT_TIMEOUT)
            if isinstance(emit, BaseException):
                raise emit
            trace.tokens.append(emit.token)
            trace.exit_layers.append(emit.exit_layer)
            trace.exit_stages.append(emit.exit_stage)
            now = time.perf_counter()
            trace.measured_latencies.append(now - t_last)
            t_last = now
            if i == max_new_tokens - 1:
                break
            position += 1
            rows, ev = embedded([emit.token], [position])
            queues[0].put(_FwdMsg(rows, [position], position, False, ev))
    finally:
        queues[0].put(_FwdMsg(None, [], -1, True, None, stop=True))
        for t in threads:
            t.join(timeout=_EMIT_TIMEOUT)
        sys.setswitchinterval(old_switch)
    for s in stages:
        if s.exception is not None:
            raise s.exception
    for s in stages:
        s.stream.synchronize()
    trace.measured_total = time.perf_counter() - t_start

    gen = len(trace.tokens)
    if gen:
        for s in stages:
            if not s.eng.kv.complete(t0 + gen - 1):
                raise ConfigError("KV fill mask incomplete after generation")
    trace.confidences = [conf_log.get(t0 - 1 + i, {}) for i in range(gen)]
    times = stage_times if stage_times is not None else default_stage_times(part)
    lat = inference_latency(trace.exit_stages, times)
    trace.latencies = lat["pipeline_per_token"]
    trace.total_latency = lat["pipeline_total"]
    trace.baseline_latency = lat["sequential_total"]
    return trace


# ---------------------------------------------------------------------------
# Reference decoding and mode comparison — eepipe/inference.py:547-613
# ---------------------------------------------------------------------------


def greedy_reference(model: EarlyExitModel, prompt, max_new_tokens, *, dtype=None, device=None):
    """Full-prefix recomputation for every token with the final head only and
    a fresh cache each step (the uncached oracle of `eepipe/inference.py
    :547-569`), run on the same kernels."""
    cfg = model.config
    prompt = [int(t) for t in prompt]
    _check_context(cfg, len(prompt) + max_new_tokens)
    final = [hd for hd in model.heads if hd.is_final]
    L = cfg.num_layers
    eng = _engine_for(model, model.params, final, cfg, range(1, L + 1), True, dtype, device)
    toks = list(prompt)
    out = []
    torch = _torch()
    with torch.cuda.device(eng.device), torch.cuda.stream(eng.stream):
        for _ in range(max_new_tokens):
            # a fresh cache and one forced full-prefix pass per token: the
            # prefill of a one-token generation
            tr = _kv_recompute(eng, model, toks, 1.0, 1, 1)
            out.append(tr.tokens[0])
            toks.append(tr.tokens[0])
    return out


def compare_modes(model: EarlyExitModel, part: StagePartition, prompts, thresholds,
                  max_new_tokens, max_deferred=4, *, dtype=None):
    """Both inference methods over the prompt set; ``divergences`` is empty
    when tokens, exit layers and confidences agree bitwise."""
    report = {"divergences": [], "runs": []}
    for p_idx, prompt in enumerate(prompts):
        for thr in thresholds:
            pipe = generate_pipeline(part, prompt, thr, max_new_tokens, dtype=dtype)
            reco = generate_kv_recompute(model, prompt, thr, max_new_tokens, max_deferred,
                                         dtype=dtype)
            problem = None
            if pipe.tokens != reco.tokens:
                problem = next(i for i, (a, b) in enumerate(zip(pipe.tokens, reco.tokens))
                               if a != b)
            elif pipe.exit_layers != reco.exit_layers:
                problem = "exit layers"
            elif pipe.confidences != reco.confidences:
                problem = "confidences"
            if problem is not None:
                report["divergences"].append({
                    "prompt": p_idx, "threshold": thr, "first_diff": problem,
                    "pipeline": pipe.tokens, "recompute": reco.tokens})
                continue
            report["runs"].append({
                "prompt": p_idx, "threshold": thr, "tokens": list(pipe.tokens),
                "mean_exit_layer": pipe.mean_exit_layer,
                "pipeline_latency": pipe.total_latency, "pipeline_speedup": pipe.speedup,
                "recompute_latency": reco.total_latency, "recompute_speedup": reco.speedup})
    return report


# ---------------------------------------------------------------------------
# Parity/debug helpers (used by tests and the smoke check)
# ---------------------------------------------------------------------------


def prefill_taps(model: EarlyExitModel, tokens, *, dtype=None, device=None):
    """Hidden states of every prompt row at every tap 0..L (a fresh cache),
    as float32 numpy arrays — the GPU counterpart of running `_layer_step`
    layer by layer over a prompt."""
    torch = _torch()
    cfg = model.config
    L = cfg.num_layers
    eng = _engine_for(model, model.params, model.heads, cfg, range(1, L + 1), True, dtype, device)
    n = len(tokens)
    taps = []
    with torch.cuda.device(eng.device), torch.cuda.stream(eng.stream):
        eng.kv.reset()
        eng._grow(n)
        eng.embed_rows(list(tokens), range(n), 0)
        eng.upload_ctrl(list(range(n)))
        taps.append(eng.x[:n].cpu().numpy().copy())
        for l in range(1, L + 1):
            eng.run_layers(l - 1, l, n, [n], n - 1, 0, prefill=True)
            eng.kv.mark_written(l - 1, l, list(range(n)), n - 1)
            taps.append(eng.x[:n].cpu().numpy().copy())
    return taps


def head_logits(model: EarlyExitModel, head_key, rows, threshold=1.0, *, dtype=None, device=None):
    """Run one head's fused kernel on given float32 hidden rows (m <= 16)
    with the debug logits dump enabled.  Returns (logits (m, V) float32,
    tokens, confidences, fires) as numpy arrays."""
    torch = _torch()
    cfg = model.config
    L = cfg.num_layers
    eng = _engine_for(model, model.params, model.heads, cfg, range(1, L + 1), True, dtype, device)
    hi = next(i for i, e in enumerate(eng.heads) if e.desc.key == head_key)
    e = eng.heads[hi]
    rows = np.asarray(rows, dtype=np.float32).reshape(-1, cfg.hidden_dim)
    m = rows.shape[0]
    if m > _HEAD_MAX_ROWS:
        raise ConfigError(f"at most {_HEAD_MAX_ROWS} rows per head call")
    with torch.cuda.device(eng.device), torch.cuda.stream(eng.stream):
        eng._grow(m)
        eng.x[:m].copy_(torch.from_numpy(rows))
        eng.upload_ctrl(list(range(m)))
        dbg = torch.zeros((m, e.V), dtype=torch.float32, device=eng.device)
        eng.eval_head(e, eng.ctrl_ptr(0), m, threshold, 0, logits_dbg=dbg)
        eng.fetch_results(1)
        out = dbg.cpu().numpy()
    return (out, eng.h_tok[0, :m].copy(), eng.h_conf[0, :m].copy(),
            eng.h_fire[0, :m].astype(bool))
