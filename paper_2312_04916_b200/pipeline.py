"""1F1B pipeline-parallel early-exit training.

Mirrors `eepipe/pipeline.py` (the reference simulates stages with threads
and `queue.Queue`s):

* each stage follows the structural 1F1B action list
  (`schedule.regular_actions`, eepipe/schedule.py:170-179): warm-up
  ``min(P-s, M)`` forwards, then (F, B) pairs, then the trailing backwards;
* activations x_s flow forward and the early-exit loss-backprop signals
  g_s = dL_aux/dx_s flow backward over ordered point-to-point channels; a
  stage's backward step builds the surrogate
  ``aux = sum_e w_e * CE_e + <g, x_sent>`` (eepipe/pipeline.py:195-223) by
  ``torch.autograd.backward([local_loss, x_out], [1, g])``;
* early exits are DEFERRED: their loss is formed inside the backward step
  (eepipe/pipeline.py:175-192), through the fused tcgen05 head, so no
  stage ever holds exit logits;
* gradients accumulate as raw sums over microbatches (:422-427) and tied
  replicas are summed after the iteration (`sync_tied`, :226-241).

Two transports share the same `StageWorker`:

* `run_iteration_1f1b`: one thread per stage in this process, each stage on
  its own CUDA stream / device, channels are ordered queues carrying device
  tensors (the reference's topology, on GPUs);
* `run_stage_1f1b_dist`: one process per GPU (torchrun), channels are
  `torch.distributed` point-to-point sends over NCCL (NVLink), tied-replica
  sync is an all-reduce over the holders' subgroup.  The protocol is covered
  on CPU with the gloo backend (tests/test_pipeline_dist.py).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from queue import Empty, Queue

from . import schedule as sched
from .errors import ConfigError, QueueProtocolError, ShapeError
from .model import StagePartition

_RECV_TIMEOUT = 120.0


def _torch():
    import torch
    return torch


@dataclass
class ActivationMessage:
    mb: int
    data: object


@dataclass
class GradientMessage:
    mb: int
    data: object


@dataclass(frozen=True)
class WeightSchedule:
    """Per-exit loss weights over training steps (eepipe/pipeline.py:47-84):
    ``constant`` returns ``early`` forever; ``linear`` interpolates from
    ``early`` to ``early_end`` over ``span_steps`` and clamps.  The final
    exit's weight stays fixed."""

    kind: str = "constant"
    early: tuple = ()
    early_end: tuple = ()
    span_steps: int = 0
    final_weight: float = 1.0


def weight_at_step(ws: WeightSchedule, step: int):
    if ws.kind == "constant":
        early = list(ws.early)
    elif ws.kind == "linear":
        if len(ws.early_end) != len(ws.early):
            raise ConfigError("linear schedule needs early_end for every early exit")
        frac = 1.0 if ws.span_steps <= 0 else min(max(step / ws.span_steps, 0.0), 1.0)
        early = [a + (b - a) * frac for a, b in zip(ws.early, ws.early_end)]
    else:
        raise ConfigError(f"unknown weight schedule {ws.kind!r}")
    return early + [ws.final_weight]


@dataclass
class IterationOptions:
    """eepipe/pipeline.py:164-172 (incl. ``fill_plan`` / ``fill_batch`` for
    bubble filling), plus ``hoist_exit_heads``: form a stage's exit losses
    before receiving its backward gradient (the paper's §4.2.2 Remark;
    gradients are identical either way)."""

    microbatch_size: int
    defer_exit_forward: bool = True
    weight_schedule: WeightSchedule | None = None
    step: int = 0
    hoist_exit_heads: bool = True
    fill_plan: object = None   # bubblefill.FillPlan
    fill_batch: object = None  # rows of the extra (fill) microbatches
    cost: object = None        # schedule.CostModel overriding the simulator's preset times


@dataclass
class StageMemoryCounters:
    """Per-stage memory counters (eepipe/pipeline.py:125-130).  The fused
    exit head never materialises logits, so ``peak_logit_copies`` is 0 in
    both exit-forward variants (the reference holds one (b, s, V) copy per
    deferred head evaluation, and one per in-flight microbatch when eager)."""

    stage: int
    peak_stored_microbatches: int = 0
    peak_fill_stored: int = 0
    peak_logit_copies: int = 0


@dataclass
class TrainStepReport:
    """Per-iteration record with the reference's fields
    (eepipe/pipeline.py:133-161): per-exit mean losses, per-stage gradient
    norms, wall clock, per-stage memory counters, microbatch count, per-stage
    executed (kind, microbatch) order, message counts, weights used."""

    per_exit_losses: dict = field(default_factory=dict)
    grad_norms: dict = field(default_factory=dict)
    wall_clock: dict = field(default_factory=dict)
    memory: list = field(default_factory=list)
    microbatches: int = 0
    event_log: list = field(default_factory=list)
    activation_messages: dict = field(default_factory=dict)
    gradient_messages: dict = field(default_factory=dict)
    weights_used: tuple = ()
    timeline: object = None

    def semantic_state(self):
        """Everything that must be reproducible under a fixed seed and
        schedule, wall clock excluded (eepipe/pipeline.py:146-161)."""
        return (
            tuple(sorted(self.per_exit_losses.items())),
            tuple(sorted(self.grad_norms.items())),
            tuple((m.stage, m.peak_stored_microbatches, m.peak_fill_stored, m.peak_logit_copies)
                  for m in self.memory),
            self.microbatches,
            tuple(tuple(log) for log in self.event_log),
            tuple(sorted(self.activation_messages.items())),
            tuple(sorted(self.gradient_messages.items())),
            self.weights_used,
        )

    @property
    def per_exit_loss(self):  # earlier name, kept for callers of this package
        return self.per_exit_losses

    @property
    def max_in_flight(self):
        return {m.stage: m.peak_stored_microbatches for m in self.memory}


def _grad_norm(grads):
    """L2 norm over a stage's gradient tensors: one fused multi-tensor norm
    launch and a single host read (eepipe/pipeline.py:626-631)."""
    torch = _torch()
    ts = [g.detach() for g in grads.values()]
    if not ts:
        return 0.0
    norms = torch._foreach_norm([t.float() if t.dtype != torch.float32 else t for t in ts])
    return float(torch.linalg.vector_norm(torch.stack(norms).double()))


_KIND_CODE = {"mb": 0, "p1": 1, "p2": 2}
_KIND_NAME = {v: k for k, v in _KIND_CODE.items()}


def _tag(mb):
    """Message tags: ("mb", k) regular microbatch k, ("p1", i) / ("p2", i)
    Part-1 / Part-2 fill i (eepipe/pipeline.py:86-122); a bare int is a
    regular id."""
    return ("mb", mb) if isinstance(mb, int) else tuple(mb)


class TaggedChannel:
    """In-process P2P channel with tag-addressed receive
    (eepipe/pipeline.py:86-122): messages arrive in sender order, the
    receiver may consume them slightly out of order (fills interleave with
    steady-phase traffic), so popped messages are stashed until their tag is
    requested; regular microbatch ids must arrive strictly increasing."""

    def __init__(self, name):
        self.name = name
        self.q = Queue()
        self.stash = {}
        self.last = 0
        self.count = 0

    def send(self, msg):
        """Device tensors are produced asynchronously on the sender's stream:
        the message carries an event recorded there, and the receiver's
        stream waits on it before any kernel reads the tensor."""
        self.count += 1
        ev = None
        data = getattr(msg, "data", None)
        if data is not None and getattr(data, "is_cuda", False):
            torch = _torch()
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(data.device))
        self.q.put((msg, ev))

    def _ready(self, item):
        msg, ev = item
        if ev is not None:
            torch = _torch()
            stream = torch.cuda.current_stream(msg.data.device)
            stream.wait_event(ev)
            # the sender's allocator must not recycle the block while this
            # stream still uses it
            msg.data.record_stream(stream)
        return msg

    def recv(self, tag):
        tag = _tag(tag)
        if tag in self.stash:
            return self._ready(self.stash.pop(tag))
        while True:
            try:
                item = self.q.get(timeout=_RECV_TIMEOUT)
            except Empty:
                raise QueueProtocolError(f"{self.name}: timed out waiting for message {tag}")
            if isinstance(item, BaseException):
                raise item
            got = _tag(item[0].mb)
            if got[0] == "mb":
                if got[1] <= self.last:
                    raise QueueProtocolError(f"{self.name}: microbatch ids out of order: "
                                             f"{got[1]} after {self.last}")
                self.last = got[1]
            if got == tag:
                return self._ready(item)
            self.stash[got] = item


_CTRL_GROUPS = {}


class Wire:
    """Point-to-point transport between stage processes.

    * Control words (message tags, positions, statuses) are host int64
      tensors on a gloo group: the receiver learns what comes next without a
      device-to-host copy and stream synchronisation per header.
    * Tensors go over the default group: NCCL (device memory, NVLink) on a
      multi-GPU box; with a gloo default group (CPU tests, or several stage
      processes sharing ONE GPU, which NCCL refuses) device tensors are
      staged through host memory.
    Sends are non-blocking and kept alive until `flush`."""

    def __init__(self):
        torch = _torch()
        dist = torch.distributed
        self.backend = dist.get_backend()
        self.staged = self.backend != "nccl"
        if self.backend == "gloo":
            self.ctrl = None
        else:  # every rank creates it once, in the same order (collective)
            key = id(dist.group.WORLD)
            if key not in _CTRL_GROUPS:
                _CTRL_GROUPS[key] = dist.new_group(backend="gloo")
            self.ctrl = _CTRL_GROUPS[key]
        self.pending = []

    def send_ints(self, vals, dst):
        torch = _torch()
        t = torch.tensor(list(vals), dtype=torch.int64)
        self.pending.append((torch.distributed.isend(t, dst, group=self.ctrl), t))

    def recv_ints(self, n, src):
        torch = _torch()
        t = torch.empty(n, dtype=torch.int64)
        torch.distributed.recv(t, src, group=self.ctrl)
        return t.tolist()

    def send(self, t, dst):
        torch = _torch()
        if self.staged and t.device.type == "cuda":
            t = t.to("cpu")  # waits for the producing stream: the device data is final
        t = t.contiguous()
        self.pending.append((torch.distributed.isend(t, dst), t))

    def recv(self, shape, dtype, device, src):
        """Blocking receive into a fresh tensor on ``device``, ready on the
        caller's current stream."""
        torch = _torch()
        device = torch.device(device)
        if self.staged and device.type == "cuda":
            h = torch.empty(shape, dtype=dtype)
            torch.distributed.recv(h, src)
            return h.to(device)
        t = torch.empty(shape, dtype=dtype, device=device)
        torch.distributed.recv(t, src)
        return t

    def flush(self):
        for req, _ in self.pending:
            req.wait()
        self.pending = []


class DistChannel:
    """Ordered (tag, tensor) channel between two stage processes over a
    `Wire` (tags on the gloo control group, tensors over NCCL / staged
    gloo).  Sends are non-blocking (isend), like the reference's queue puts:
    with blocking sends the 1F1B steady state would deadlock (stage s sending
    x while stage s+1 sends g back).  `flush` waits for the outstanding
    sends."""

    def __init__(self, peer, shape, dtype, device, wire=None):
        self.peer, self.shape, self.dtype, self.device = peer, tuple(shape), dtype, device
        self.wire = wire if wire is not None else Wire()
        self.last = 0
        self.count = 0
        self.stash = {}

    def send(self, msg):
        data = msg.data.contiguous()
        if tuple(data.shape) != self.shape:
            raise ShapeError(f"channel expects {self.shape}, got {tuple(data.shape)}")
        tag = _tag(msg.mb)
        self.wire.send_ints((_KIND_CODE[tag[0]], tag[1]), self.peer)
        self.wire.send(data, self.peer)
        self.count += 1

    def flush(self):
        self.wire.flush()

    def recv(self, tag):
        """Messages arrive in the sender's order (point-to-point operations
        match in order per peer); each carries its tag, so a message
        requested later than it arrives is stashed, like the reference's
        tagged queue (eepipe/pipeline.py:86-122).  Regular ids must arrive
        increasing."""
        tag = _tag(tag)
        if tag in self.stash:
            return self.stash.pop(tag)
        while True:
            code, idx = self.wire.recv_ints(2, self.peer)
            got = (_KIND_NAME[code], idx)
            if got[0] == "mb":
                if idx <= self.last:
                    raise QueueProtocolError(f"microbatch ids out of order: {idx} after {self.last}")
                self.last = idx
            data = self.wire.recv(self.shape, self.dtype, self.device, self.peer)
            msg = type("Msg", (), {"mb": got, "data": data})
            if got == tag:
                return msg
            self.stash[got] = msg


_UNSET = object()


class StageCompute:
    """Product stage compute: the stage's layers with torch autograd on its
    device and the fused tcgen05 exit heads; exit losses are formed in the
    backward step (deferred exit forward)."""

    def __init__(self, spec, cfg, model_src, weights, device=None, dtype=None, master_dtype=None):
        from .training import TrainModel
        self.spec = spec
        self.cfg = cfg
        self.tm = TrainModel(model_src, dtype=dtype, device=device, names=list(spec.params),
                             master_dtype=master_dtype)
        self.device = self.tm.device
        self.weights = weights  # by head key
        self.head_losses = {hd.key: [] for _, hd in spec.heads}

    def reset(self, weights):
        """Start a new iteration on the same device state."""
        self.weights = weights
        self.head_losses = {hd.key: [] for _, hd in self.spec.heads}
        self.tm.zero_grad()

    def forward(self, tokens_or_x, targets, grad=True):
        """``grad=False``: forward only (a Part-2 fill on a stage its
        backward does not cover, eepipe/pipeline.py:476-489)."""
        from .training import embed_tokens, run_layer
        torch = _torch()
        with torch.set_grad_enabled(grad):
            p = self.tm.compute_params()
            if self.spec.has_embedding:
                x_in = None
                x = embed_tokens(p, tokens_or_x, self.cfg.max_seq_len)
            else:
                x_in = tokens_or_x.to(self.device).detach().requires_grad_(grad)
                x = x_in
            taps = {0: x}
            for local, layer in enumerate(self.spec.layer_indices, start=1):
                x = run_layer(p, f"layer{layer}", x, self.cfg.num_heads)
                taps[local] = x
        return x, (x_in, x, taps, targets)

    def local_loss(self, state, include_final=True, record=True):
        """Weighted sum of this stage's exit losses.  Part-1 fills leave the
        final head out and no fill records losses (eepipe/pipeline.py:456-474)."""
        import numpy as np
        from .training import head_loss
        torch = _torch()
        _, _, taps, targets = state
        from .training import _check_ids, to_device_async
        heads = [(local, hd) for local, hd in self.spec.heads if include_final or not hd.is_final]
        if not heads:
            return None
        _check_ids(targets, self.cfg.vocab_size, "target")
        targets = to_device_async(np.ascontiguousarray(targets), self.device)
        total = None
        params = self.tm.compute_params()
        for local, hd in heads:
            ce = head_loss(params, hd, taps[local], targets, self.cfg.num_heads, validated=True)
            if record:
                self.head_losses[hd.key].append(ce.detach())  # read after the iteration (no sync)
            term = ce * self.weights[hd.key]
            total = term if total is None else total + term
        return total

    def backward(self, state, g, loss=_UNSET, include_final=True, record=True):
        """``loss``: the stage's local exit loss when the worker already
        formed it (hoisted ahead of the gradient receive); otherwise it is
        formed here (deferred exit forward, eepipe/pipeline.py:393-412)."""
        torch = _torch()
        x_in, x_out, _, _ = state
        if loss is _UNSET:
            loss = self.local_loss(state, include_final, record)
        if g is None:
            if loss is None:
                raise ConfigError("a stage must have a local loss or a received gradient")
            loss.backward()
        else:
            if tuple(g.shape) != tuple(x_out.shape):
                raise ShapeError(f"gradient shape {tuple(g.shape)} does not match activation "
                                 f"{tuple(x_out.shape)}")
            # aux = L_local + <g, x_out>  (eepipe/pipeline.py:195-223)
            outs, grads = [x_out], [g.to(x_out.dtype)]
            if loss is not None:
                outs.insert(0, loss)
                grads.insert(0, torch.ones_like(loss))
            torch.autograd.backward(outs, grads)
        self.tm.accumulate_grads()  # mixed precision: fold into float32 sums (one launch)
        return None if x_in is None else x_in.grad


@dataclass
class _FillContext:
    """Per-iteration bubble-fill geometry (eepipe/pipeline.py:527-535):
    truncated Part-1 depths (None = skipped) and the stage sets each Part-2
    microbatch's backward covers."""

    part1_depths: list = field(default_factory=list)
    part2_covered: list = field(default_factory=list)


class StageWorker:
    """Executes one stage's action list (eepipe/pipeline.py:301-527): the
    1F1B order, plus bubble-fill microbatches when ``fill`` is given."""

    def __init__(self, index, num_stages, num_mb, compute, data, fwd_in, fwd_out, bwd_in,
                 bwd_out, hoist_exits=True, actions=None, fill=None):
        self.index, self.P, self.M = index, num_stages, num_mb
        self.compute = compute
        self.data = data  # regular k -> (tokens, targets); ("p1"|"p2", i) -> fill rows
        self.fwd_in, self.fwd_out, self.bwd_in, self.bwd_out = fwd_in, fwd_out, bwd_in, bwd_out
        self.hoist_exits = hoist_exits and hasattr(compute, "local_loss")
        self.actions = actions if actions is not None else sched.regular_actions(
            num_stages, num_mb, index)
        self.fill = fill
        self.state = {}
        self.event_log = []
        self.wall = {"F": 0.0, "B": 0.0}
        self.in_flight = 0
        self.max_in_flight = 0
        self.fill_stored = 0
        self.max_fill_stored = 0
        self.exception = None

    def run(self):
        try:
            for kind, i in self.actions:
                t = time.perf_counter()
                if kind == sched.FWD:
                    self._forward(("mb", i))
                elif kind == sched.BWD:
                    self._backward(("mb", i))
                elif kind == sched.FILL1_FWD:
                    d = self.fill.part1_depths[i - 1]
                    self._forward(("p1", i), send=self.index < d)
                elif kind == sched.FILL1_BWD:
                    d = self.fill.part1_depths[i - 1]
                    self._backward(("p1", i), recv=self.index < d, send=self.index > 1,
                                   include_final=False)
                elif kind == sched.FILL2_FWD:
                    covered = self.index in self.fill.part2_covered[i - 1]
                    self._forward(("p2", i), keep=covered)
                elif kind == sched.FILL2_BWD:
                    deepest = min(self.fill.part2_covered[i - 1])
                    self._backward(("p2", i), send=self.index > deepest)
                else:
                    raise ConfigError(f"unknown action {kind!r}")
                self.wall["F" if kind in sched.FWD_KINDS else "B"] += time.perf_counter() - t
                self.event_log.append((kind, i))
            if self.state:
                raise QueueProtocolError(
                    f"stage {self.index} finished with unconsumed activations")
        except BaseException as exc:  # surfaced by the coordinator
            self.exception = exc
            for ch in (self.fwd_out, self.bwd_out):
                if isinstance(ch, TaggedChannel):
                    ch.q.put(exc)

    def _rows(self, tag):
        return self.data[tag[1]] if tag[0] == "mb" else self.data[tag]

    def _count(self, tag, delta):
        if tag[0] == "mb":
            self.in_flight += delta
            self.max_in_flight = max(self.max_in_flight, self.in_flight)
        else:
            self.fill_stored += delta
            self.max_fill_stored = max(self.max_fill_stored, self.fill_stored)

    def _forward(self, tag, send=True, keep=True):
        """``keep=False``: forward only, nothing stored (a Part-2 fill on an
        uncovered stage)."""
        tokens, targets = self._rows(tag)
        src = tokens if self.fwd_in is None else self.fwd_in.recv(tag).data
        x_out, st = self.compute.forward(src, targets) if keep else \
            self.compute.forward(src, targets, grad=False)
        if keep:
            self.state[tag] = st
            self._count(tag, 1)
        if send and self.fwd_out is not None:
            self.fwd_out.send(ActivationMessage(tag, x_out.detach()))

    def _backward(self, tag, recv=None, send=None, include_final=True):
        """``recv`` / ``send``: whether the downstream gradient arrives /
        the input gradient leaves (default: whenever the neighbour exists).
        Fills record no losses."""
        st = self.state.pop(tag)
        recv = self.bwd_in is not None if recv is None else recv
        send = self.bwd_out is not None if send is None else send
        record = tag[0] == "mb"
        if self.hoist_exits and recv:
            # the paper's §4.2.2 Remark (modelled only by the reference,
            # eepipe/schedule.py:491-502): form the stage's exit losses — with
            # the fused head that is the whole exit forward AND backward —
            # before waiting for the downstream gradient, so the exit work
            # overlaps the pipeline's communication instead of following it
            loss = self.compute.local_loss(st, include_final, record) if not (
                include_final and record) else self.compute.local_loss(st)
            g = self.bwd_in.recv(tag).data
            g_in = self.compute.backward(st, g, loss)
        else:
            g = self.bwd_in.recv(tag).data if recv else None
            g_in = self.compute.backward(st, g) if (include_final and record) else \
                self.compute.backward(st, g, include_final=include_final, record=record)
        self._count(tag, -1)
        if send:
            if g_in is None:
                raise ConfigError("stored input activation received no gradient")
            self.bwd_out.send(GradientMessage(tag, g_in.detach()))


def _resolve_weights(heads, options):
    if options.weight_schedule is not None:
        w = weight_at_step(options.weight_schedule, options.step)
        if len(w) != len(heads):
            raise ConfigError(f"schedule yields {len(w)} weights for {len(heads)} exits")
        return list(w)
    return [hd.loss_weight for hd in heads]


def _split(batch, mb_size):
    import numpy as np
    batch = np.asarray(batch)
    if batch.ndim != 2 or batch.shape[0] % mb_size:
        raise ConfigError("batch does not divide into microbatches")
    M = batch.shape[0] // mb_size
    return M, {k + 1: (batch[k * mb_size:(k + 1) * mb_size, :-1],
                       batch[k * mb_size:(k + 1) * mb_size, 1:]) for k in range(M)}


def sync_tied(per_stage_grads, tied_replicas=None):
    """Sum replica gradients by canonical name (eepipe/pipeline.py:226-241);
    tensors may live on different devices (summed on the first holder's)."""
    merged = {}
    for stage_map in per_stage_grads:
        for name, g in stage_map.items():
            if name in merged:
                if merged[name].shape != g.shape:
                    raise ShapeError(f"replica shape mismatch for {name}")
                merged[name] = merged[name] + g.to(merged[name].device)
            else:
                merged[name] = g
    return merged


_STAGE_STREAMS = {}


def _stage_stream(device, stage):
    """One persistent CUDA stream per (device, stage): per-stream scratch
    (workspaces, upload rings) is then allocated once, not per iteration."""
    torch = _torch()
    dev = torch.device(device)
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), stage)
    st = _STAGE_STREAMS.get(key)
    if st is None:
        st = _STAGE_STREAMS[key] = torch.cuda.Stream(device)
    return st


def cost_model_from_partition(part: StagePartition, num_microbatches: int,
                              microbatch_size: int, seq_len: int, base=None):
    """The schedule cost model of a partition (`eepipe/pipeline.py:262-285`):
    early exits per stage from the partition, the preset (or ``base``)
    step times."""
    cfg = part.config
    counts = [0] * part.num_stages
    for st in part.stages:
        counts[st.index - 1] = sum(1 for _, hd in st.heads if not hd.is_final)
    kw = dict(num_stages=part.num_stages, num_microbatches=num_microbatches,
              exit_counts=tuple(counts), seq_len=seq_len, microbatch_size=microbatch_size,
              vocab_size=cfg.vocab_size, hidden_dim=cfg.hidden_dim,
              layers_per_stage=cfg.num_layers // part.num_stages)
    if base is not None:
        kw.update(fwd_time=base.fwd_time, bwd_time=base.bwd_time,
                  exit_fwd_time=base.exit_fwd_time, exit_bwd_time=base.exit_bwd_time,
                  embed_fwd_time=base.embed_fwd_time, p2p_latency=base.p2p_latency)
    return sched.CostModel(**kw)


def apply_fill(plan, part: StagePartition, num_microbatches: int):
    """Validate a fill plan against a partition; returns (truncated Part-1
    depths, FillRescale) (eepipe/pipeline.py:244-259).  Tied parameters
    across stages reject the plan."""
    from .bubblefill import fill_rescale, truncated_part1_depths
    if part.tied_replicas:
        raise ConfigError("bubble filling requires untied parameters across stages; "
                          f"tied: {sorted(part.tied_replicas)}")
    if plan.num_stages != part.num_stages:
        raise ConfigError("fill plan stage count does not match the partition")
    exit_stages = part.exit_stages()
    return (truncated_part1_depths(plan, exit_stages),
            fill_rescale(plan, exit_stages, num_microbatches))


def _assign_fill_data(data, row_len, options: IterationOptions, depths):
    """Fill microbatches take consecutive microbatch-size slices of
    ``fill_batch``: executed Part-1 fills first, then Part-2
    (eepipe/pipeline.py:658-680)."""
    import numpy as np
    plan = options.fill_plan
    executed = [i for i, d in enumerate(depths, 1) if d is not None]
    needed = len(executed) + len(plan.part2_bwd_depths)
    fb = options.fill_batch
    if fb is None and needed:
        raise ConfigError("fill plan is active but no fill_batch was provided")
    fb = np.asarray(fb) if fb is not None else np.empty((0, row_len), dtype=np.int64)
    mbs = options.microbatch_size
    if fb.ndim != 2 or fb.shape[0] != needed * mbs or fb.shape[1] != row_len:
        raise ConfigError(f"fill_batch must hold {needed} microbatches of the batch row length")
    k = 0
    for tag in [("p1", i) for i in executed] + [("p2", i) for i in
                                                 range(1, len(plan.part2_bwd_depths) + 1)]:
        rows = fb[k * mbs:(k + 1) * mbs]
        data[tag] = (rows[:, :-1], rows[:, 1:])
        k += 1


_STAGE_EXECUTORS = {}


def _stage_executor(device, stage):
    """One persistent worker thread per (device, stage): library state that
    is per host thread (the cuDNN handle and its attention execution-plan
    cache) survives across iterations — a fresh thread per iteration rebuilt
    the SDPA plan, a ~50 ms host stall at the first attention of every
    step."""
    from concurrent.futures import ThreadPoolExecutor
    key = (str(device), stage)
    ex = _STAGE_EXECUTORS.get(key)
    if ex is None:
        ex = _STAGE_EXECUTORS[key] = ThreadPoolExecutor(max_workers=1,
                                                        thread_name_prefix=f"stage-{stage}")
    return ex


@dataclass
class _IterationPlan:
    M: int
    data: dict
    all_heads: list
    weights: list
    wmap: dict
    fill: object
    rescale: object
    depths: list
    plan: object
    timeline: object
    n_fill: int


def _plan_iteration(part: StagePartition, batch, options: IterationOptions) -> _IterationPlan:
    """Everything both executors derive before running: microbatches, head
    weights (Part-1-rescaled), the fill geometry and data, and the simulated
    timeline whose per-stage order the workers execute
    (eepipe/pipeline.py:537-590)."""
    import numpy as np
    P = part.num_stages
    M, data = _split(batch, options.microbatch_size)
    all_heads = [hd for st in part.stages for _, hd in st.heads]
    all_heads.sort(key=lambda hd: (hd.layer_index, hd.is_final))
    weights = _resolve_weights(all_heads, options)
    wmap = {hd.key: w for hd, w in zip(all_heads, weights)}
    # bubble filling (eepipe/pipeline.py:566-580): Part-1-sampled exit losses
    # get their weight scaled in every microbatch, Part-2-covered stages
    # their accumulated gradient
    fill, rescale, depths = None, None, []
    plan = options.fill_plan
    if plan is not None and not plan.empty:
        if not options.defer_exit_forward:
            raise ConfigError("bubble filling requires the deferred-exit variant")
        if M < P:
            raise ConfigError("bubble filling needs at least P microbatches")
        depths, rescale = apply_fill(plan, part, M)
        covered = [set(range(P - r + 1, P + 1)) for r in plan.part2_bwd_depths]
        fill = _FillContext(list(depths), covered)
        _assign_fill_data(data, np.asarray(batch).shape[1], options, depths)
        for hd in all_heads:
            if not hd.is_final:
                wmap[hd.key] = wmap[hd.key] * rescale.weight_scale_for(part.stage_of_head(hd.key))
    # the per-stage action order is the simulated timeline's
    # (eepipe/pipeline.py:553-557, 587): the 1F1B lists, with fills placed
    # where the cost model finds the bubbles
    seq_len = int(np.asarray(batch).shape[1]) - 1
    timeline = sched.simulate(
        cost_model_from_partition(part, M, options.microbatch_size, seq_len, options.cost),
        "deferred-exit" if options.defer_exit_forward else "eager-exit",
        plan if fill is not None else None)
    n_fill = (sum(1 for d in depths if d is not None) + len(plan.part2_bwd_depths)
              if fill is not None else 0)
    return _IterationPlan(M, data, all_heads, weights, wmap, fill, rescale, depths, plan,
                          timeline, n_fill)


def run_iteration_1f1b(part: StagePartition, batch, options: IterationOptions, model=None,
                       devices=None, dtype=None, master_dtype=None, stage_computes=None,
                       compute_factory=None):
    """One 1F1B iteration over the partition, one thread per stage
    (eepipe/pipeline.py:537-644).  ``model`` is the EarlyExitModel the stage
    weights come from (the partition's own copies are used when omitted).
    ``master_dtype=torch.float32`` accumulates gradients in float32
    (`TrainModel` mixed mode).  ``stage_computes``: a list that keeps the
    per-stage device state across iterations (filled on the first call,
    reused — gradients zeroed, weights as the optimizer left them — after).
    ``compute_factory(spec, cfg, wmap)`` overrides the stage compute (CPU
    protocol tests).  Returns (merged gradient map by name, TrainStepReport)."""
    P = part.num_stages
    it = _plan_iteration(part, batch, options)
    M, data, all_heads, weights, wmap = it.M, it.data, it.all_heads, it.weights, it.wmap
    fill, rescale, depths, plan, timeline = it.fill, it.rescale, it.depths, it.plan, it.timeline
    devices = devices or ["cuda:0"] * P
    src = model
    fwd = [TaggedChannel(f"act {s}->{s + 1}") for s in range(1, P)]
    bwd = [TaggedChannel(f"grad {s + 1}->{s}") for s in range(1, P)]
    workers = []
    reuse = stage_computes is not None and len(stage_computes) == P
    for s, spec in enumerate(part.stages, start=1):
        if compute_factory is not None:
            comp = compute_factory(spec, part.config, wmap)
        elif reuse:
            comp = stage_computes[s - 1]
            comp.reset(wmap)
        else:
            holder = src if src is not None else _SpecModel(part, spec)
            comp = StageCompute(spec, part.config, holder, wmap, devices[(s - 1) % len(devices)],
                                dtype, master_dtype)
            if stage_computes is not None:
                stage_computes.append(comp)
        workers.append(StageWorker(s, P, M, comp, data,
                                   fwd[s - 2] if s > 1 else None, fwd[s - 1] if s < P else None,
                                   bwd[s - 1] if s < P else None, bwd[s - 2] if s > 1 else None,
                                   options.hoist_exit_heads, actions=timeline.order(s),
                                   fill=fill))
    torch = _torch()
    # the stage streams start after everything the caller queued on its own
    # stream: the gradient zeroing of comp.reset above and the previous
    # step's optimizer update (which rewrites the bf16 weights the stages read)
    ready = {}
    for w in workers:
        dev = torch.device(w.compute.device)
        if dev.type == "cuda" and str(dev) not in ready:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dev))
            ready[str(dev)] = ev

    def target(w):
        dev = torch.device(w.compute.device)
        if dev.type != "cuda":
            w.run()
            return
        st = _stage_stream(dev, w.index)
        st.wait_event(ready[str(dev)])
        with torch.cuda.device(dev), torch.cuda.stream(st):
            w.run()
            from .training import join_wgrad
            join_wgrad(dev)
            torch.cuda.current_stream(dev).synchronize()

    t_start = time.perf_counter()
    import sys
    old_switch = sys.getswitchinterval()
    if P > 1:  # several launch-bound stage threads: hand the GIL over quickly
        sys.setswitchinterval(5e-5)
    try:
        futures = [_stage_executor(torch.device(w.compute.device), w.index).submit(target, w)
                   for w in workers]
        for f in futures:
            f.result(timeout=_RECV_TIMEOUT * 2)
    finally:
        sys.setswitchinterval(old_switch)
    elapsed = time.perf_counter() - t_start
    for w in workers:
        if w.exception is not None:
            raise w.exception
    per_stage = [w.compute.tm.grads() if compute_factory is None else w.compute.grads()
                 for w in workers]
    if rescale is not None:
        for w, g in zip(workers, per_stage):
            gs = rescale.grad_scale_for(w.index)
            if gs != 1.0:
                for t in g.values():
                    t.mul_(gs)
    merged = sync_tied(per_stage, part.tied_replicas)
    report = TrainStepReport(weights_used=tuple(weights), microbatches=M + it.n_fill,
                             timeline=timeline)
    for w, g in zip(workers, per_stage):
        report.event_log.append(list(w.event_log))
        report.memory.append(StageMemoryCounters(w.index, w.max_in_flight, w.max_fill_stored))
        report.grad_norms[w.index] = _grad_norm(g)
        report.activation_messages[w.index] = w.fwd_out.count if w.fwd_out is not None else 0
        report.gradient_messages[w.index] = w.bwd_out.count if w.bwd_out is not None else 0
    for hd in all_heads:
        vals = [v for w in workers for v in w.compute.head_losses.get(hd.key, [])]
        report.per_exit_losses[hd.key] = sum(float(v) for v in vals) / len(vals)
    report.wall_clock = {"forward": sum(w.wall["F"] for w in workers),
                         "backward": sum(w.wall["B"] for w in workers), "total": elapsed}
    return merged, report


class _SpecModel:
    """Adapter exposing a stage's own parameter copies as a model source."""

    def __init__(self, part, spec):
        self.config = part.config
        self.params = spec.params
        self.heads = [hd for _, hd in spec.heads]


def run_stage_1f1b_dist(part: StagePartition, batch, options: IterationOptions, model=None,
                        compute_factory=None, dtype=None):
    """The calling rank's stage of a distributed 1F1B iteration (one process
    per stage; rank r runs stage r+1).  Activations / gradients travel by
    `torch.distributed` P2P (NCCL over NVLink on GPUs); tied replicas are
    summed with an all-reduce over their holders.  ``compute_factory(spec,
    cfg, wmap)`` overrides the stage compute (tests use a CPU one under
    gloo).  Returns (this stage's gradient map, partial report)."""
    torch = _torch()
    dist = torch.distributed
    rank, world = dist.get_rank(), dist.get_world_size()
    P = part.num_stages
    if world != P:
        raise ConfigError(f"{world} ranks for {P} stages")
    s = rank + 1
    spec = part.stages[rank]
    it = _plan_iteration(part, batch, options)
    M, data, weights, wmap = it.M, it.data, it.weights, it.wmap
    if compute_factory is None:
        dev = torch.device("cuda", torch.cuda.current_device())
        comp = StageCompute(spec, part.config, model if model is not None else _SpecModel(part, spec),
                            wmap, dev, dtype)
        act_dtype = comp.tm.dtype
    else:
        comp = compute_factory(spec, part.config, wmap)
        dev, act_dtype = comp.device, comp.act_dtype
    mb_size = options.microbatch_size
    seq = data[1][0].shape[1]
    shape = (mb_size, seq, part.config.hidden_dim)
    wire = Wire()
    fwd_in = DistChannel(rank - 1, shape, act_dtype, dev, wire) if s > 1 else None
    fwd_out = DistChannel(rank + 1, shape, act_dtype, dev, wire) if s < P else None
    bwd_in = DistChannel(rank + 1, shape, act_dtype, dev, wire) if s < P else None
    bwd_out = DistChannel(rank - 1, shape, act_dtype, dev, wire) if s > 1 else None
    w = StageWorker(s, P, M, comp, data, fwd_in, fwd_out, bwd_in, bwd_out,
                    options.hoist_exit_heads, actions=it.timeline.order(s), fill=it.fill)
    if dev.type == "cuda":
        with torch.cuda.device(dev):
            w.run()
            from .training import join_wgrad
            join_wgrad(dev)
            torch.cuda.current_stream(dev).synchronize()
    else:
        w.run()
    wire.flush()
    if w.exception is not None:
        raise w.exception
    grads = comp.tm.grads() if compute_factory is None else comp.grads()
    if it.rescale is not None and it.rescale.grad_scale_for(s) != 1.0:
        for t in grads.values():
            t.mul_(it.rescale.grad_scale_for(s))
    # tied replicas: all-reduce(sum) over the holders (every rank joins the
    # group creation; only holders take part in the reduction)
    for name, holders in sorted(part.tied_replicas.items()):
        group = dist.new_group([h - 1 for h in holders])
        if s in holders:
            g = grads[name]
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
    # this rank's view: its own stage's entries (event_log[s-1], memory[0])
    report = TrainStepReport(weights_used=tuple(weights), microbatches=M + it.n_fill,
                             timeline=it.timeline)
    report.event_log = [[] for _ in range(P)]
    report.event_log[s - 1] = list(w.event_log)
    report.memory = [StageMemoryCounters(s, w.max_in_flight, w.max_fill_stored)]
    report.wall_clock = {"forward": w.wall["F"], "backward": w.wall["B"],
                         "total": w.wall["F"] + w.wall["B"]}
    for key, vals in comp.head_losses.items():
        report.per_exit_losses[key] = sum(float(v) for v in vals) / len(vals)
    report.activation_messages[s] = fwd_out.count if fwd_out is not None else 0
    report.gradient_messages[s] = bwd_out.count if bwd_out is not None else 0
    return grads, report
