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

import threading
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
    """eepipe/pipeline.py:164-172, plus ``hoist_exit_heads``: form a stage's
    exit losses before receiving its backward gradient (the paper's §4.2.2
    Remark; gradients are identical either way)."""

    microbatch_size: int
    defer_exit_forward: bool = True
    weight_schedule: WeightSchedule | None = None
    step: int = 0
    hoist_exit_heads: bool = True


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


class TaggedChannel:
    """Ordered in-process P2P channel; regular microbatch ids must arrive in
    strictly increasing order (eepipe/pipeline.py:87-122)."""

    def __init__(self, name):
        self.name = name
        self.q = Queue()
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

    def recv(self, expect_mb):
        try:
            item = self.q.get(timeout=_RECV_TIMEOUT)
        except Empty:
            raise QueueProtocolError(f"{self.name}: timed out waiting for microbatch {expect_mb}")
        if isinstance(item, BaseException):
            raise item
        msg, ev = item
        if msg.mb != expect_mb or msg.mb <= self.last:
            raise QueueProtocolError(
                f"{self.name}: expected microbatch {expect_mb}, got {msg.mb} (last {self.last})")
        self.last = msg.mb
        if ev is not None:
            torch = _torch()
            stream = torch.cuda.current_stream(msg.data.device)
            stream.wait_event(ev)
            # the sender's allocator must not recycle the block while this
            # stream still uses it
            msg.data.record_stream(stream)
        return msg


class DistChannel:
    """torch.distributed P2P channel carrying (mb id header, tensor) pairs in
    order between two ranks (NCCL over NVLink on GPUs, gloo on CPU).  Sends
    are non-blocking (isend), like the reference's queue puts: with blocking
    sends the 1F1B steady state would deadlock (stage s sending x while
    stage s+1 sends g back).  `flush` waits for the outstanding sends."""

    def __init__(self, peer, shape, dtype, device, group=None):
        self.peer, self.shape, self.dtype, self.device = peer, tuple(shape), dtype, device
        self.group = group
        self.last = 0
        self.count = 0
        self.pending = []

    def send(self, msg):
        torch = _torch()
        dist = torch.distributed
        data = msg.data.contiguous()
        if tuple(data.shape) != self.shape:
            raise ShapeError(f"channel expects {self.shape}, got {tuple(data.shape)}")
        hdr = torch.tensor([msg.mb], dtype=torch.int64, device=self.device)
        # keep the tensors alive until their sends complete
        self.pending.append((dist.isend(hdr, self.peer, group=self.group), hdr))
        self.pending.append((dist.isend(data, self.peer, group=self.group), data))
        self.count += 1

    def flush(self):
        for req, _ in self.pending:
            req.wait()
        self.pending = []

    def recv(self, expect_mb):
        torch = _torch()
        dist = torch.distributed
        hdr = torch.empty(1, dtype=torch.int64, device=self.device)
        dist.recv(hdr, self.peer, group=self.group)
        mb = int(hdr.item())
        if mb != expect_mb or mb <= self.last:
            raise QueueProtocolError(f"expected microbatch {expect_mb}, got {mb} (last {self.last})")
        self.last = mb
        data = torch.empty(self.shape, dtype=self.dtype, device=self.device)
        dist.recv(data, self.peer, group=self.group)
        return type("Msg", (), {"mb": mb, "data": data})


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

    def forward(self, tokens_or_x, targets):
        from .training import embed_tokens, run_layer
        p = self.tm.compute_params()
        if self.spec.has_embedding:
            x_in = None
            x = embed_tokens(p, tokens_or_x, self.cfg.max_seq_len)
        else:
            x_in = tokens_or_x.to(self.device).detach().requires_grad_()
            x = x_in
        taps = {0: x}
        for local, layer in enumerate(self.spec.layer_indices, start=1):
            x = run_layer(p, f"layer{layer}", x, self.cfg.num_heads)
            taps[local] = x
        return x, (x_in, x, taps, targets)

    def local_loss(self, state):
        import numpy as np
        from .training import head_loss
        torch = _torch()
        _, _, taps, targets = state
        from .training import _check_ids, to_device_async
        _check_ids(targets, self.cfg.vocab_size, "target")
        targets = to_device_async(np.ascontiguousarray(targets), self.device)
        total = None
        params = self.tm.compute_params()
        for local, hd in self.spec.heads:
            ce = head_loss(params, hd, taps[local], targets, self.cfg.num_heads, validated=True)
            self.head_losses[hd.key].append(ce.detach())  # read after the iteration (no sync)
            term = ce * self.weights[hd.key]
            total = term if total is None else total + term
        return total

    def backward(self, state, g, loss=_UNSET):
        """``loss``: the stage's local exit loss when the worker already
        formed it (hoisted ahead of the gradient receive); otherwise it is
        formed here (deferred exit forward, eepipe/pipeline.py:393-412)."""
        torch = _torch()
        x_in, x_out, _, _ = state
        if loss is _UNSET:
            loss = self.local_loss(state)
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


class StageWorker:
    """Executes one stage's 1F1B action list (eepipe/pipeline.py:301-527)."""

    def __init__(self, index, num_stages, num_mb, compute, data, fwd_in, fwd_out, bwd_in,
                 bwd_out, hoist_exits=True):
        self.index, self.P, self.M = index, num_stages, num_mb
        self.compute = compute
        self.data = data  # mb -> (tokens, targets)
        self.fwd_in, self.fwd_out, self.bwd_in, self.bwd_out = fwd_in, fwd_out, bwd_in, bwd_out
        self.hoist_exits = hoist_exits and hasattr(compute, "local_loss")
        self.state = {}
        self.event_log = []
        self.wall = {"F": 0.0, "B": 0.0}
        self.in_flight = 0
        self.max_in_flight = 0
        self.exception = None

    def run(self):
        try:
            for kind, mb in sched.regular_actions(self.P, self.M, self.index):
                t = time.perf_counter()
                if kind == sched.FWD:
                    self._forward(mb)
                else:
                    self._backward(mb)
                self.wall[kind] += time.perf_counter() - t
                self.event_log.append((kind, mb))
        except BaseException as exc:  # surfaced by the coordinator
            self.exception = exc
            for ch in (self.fwd_out, self.bwd_out):
                if isinstance(ch, TaggedChannel):
                    ch.q.put(exc)

    def _forward(self, mb):
        tokens, targets = self.data[mb]
        src = tokens if self.fwd_in is None else self.fwd_in.recv(mb).data
        x_out, st = self.compute.forward(src, targets)
        self.state[mb] = st
        self.in_flight += 1
        self.max_in_flight = max(self.max_in_flight, self.in_flight)
        if self.fwd_out is not None:
            self.fwd_out.send(ActivationMessage(mb, x_out.detach()))

    def _backward(self, mb):
        st = self.state.pop(mb)
        if self.hoist_exits and self.bwd_in is not None:
            # the paper's §4.2.2 Remark (modelled only by the reference,
            # eepipe/schedule.py:491-502): form the stage's exit losses — with
            # the fused head that is the whole exit forward AND backward —
            # before waiting for the downstream gradient, so the exit work
            # overlaps the pipeline's communication instead of following it
            loss = self.compute.local_loss(st)
            g = self.bwd_in.recv(mb).data
            g_in = self.compute.backward(st, g, loss)
        else:
            g = None if self.bwd_in is None else self.bwd_in.recv(mb).data
            g_in = self.compute.backward(st, g)
        self.in_flight -= 1
        if self.bwd_out is not None:
            if g_in is None:
                raise ConfigError("stored input activation received no gradient")
            self.bwd_out.send(GradientMessage(mb, g_in.detach()))


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
    key = (str(device), stage)
    st = _STAGE_STREAMS.get(key)
    if st is None:
        st = _STAGE_STREAMS[key] = torch.cuda.Stream(device)
    return st


def run_iteration_1f1b(part: StagePartition, batch, options: IterationOptions, model=None,
                       devices=None, dtype=None, master_dtype=None, stage_computes=None):
    """One 1F1B iteration over the partition, one thread per stage
    (eepipe/pipeline.py:537-644).  ``model`` is the EarlyExitModel the stage
    weights come from (the partition's own copies are used when omitted).
    ``master_dtype=torch.float32`` accumulates gradients in float32
    (`TrainModel` mixed mode).  ``stage_computes``: a list that keeps the
    per-stage device state across iterations (filled on the first call,
    reused — gradients zeroed, weights as the optimizer left them — after).
    Returns (merged gradient map by name, TrainStepReport)."""
    P = part.num_stages
    M, data = _split(batch, options.microbatch_size)
    all_heads = [hd for st in part.stages for _, hd in st.heads]
    all_heads.sort(key=lambda hd: (hd.layer_index, hd.is_final))
    weights = _resolve_weights(all_heads, options)
    wmap = {hd.key: w for hd, w in zip(all_heads, weights)}
    devices = devices or ["cuda:0"] * P
    src = model
    fwd = [TaggedChannel(f"act {s}->{s + 1}") for s in range(1, P)]
    bwd = [TaggedChannel(f"grad {s + 1}->{s}") for s in range(1, P)]
    workers = []
    reuse = stage_computes is not None and len(stage_computes) == P
    for s, spec in enumerate(part.stages, start=1):
        if reuse:
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
                                   options.hoist_exit_heads))
    torch = _torch()

    def target(w):
        dev = w.compute.device
        with torch.cuda.device(dev), torch.cuda.stream(_stage_stream(dev, w.index)):
            w.run()
            torch.cuda.current_stream(dev).synchronize()

    threads = [threading.Thread(target=target, args=(w,), daemon=True, name=f"stage-{w.index}")
               for w in workers]
    t_start = time.perf_counter()
    import sys
    old_switch = sys.getswitchinterval()
    if P > 1:  # several launch-bound stage threads: hand the GIL over quickly
        sys.setswitchinterval(5e-5)
    try:
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=_RECV_TIMEOUT * 2)
    finally:
        sys.setswitchinterval(old_switch)
    elapsed = time.perf_counter() - t_start
    for w in workers:
        if w.exception is not None:
            raise w.exception
    per_stage = [w.compute.tm.grads() for w in workers]
    merged = sync_tied(per_stage, part.tied_replicas)
    report = TrainStepReport(weights_used=tuple(weights), microbatches=M)
    for w, g in zip(workers, per_stage):
        report.event_log.append(list(w.event_log))
        report.memory.append(StageMemoryCounters(w.index, w.max_in_flight))
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
    M, data = _split(batch, options.microbatch_size)
    all_heads = sorted([hd for st in part.stages for _, hd in st.heads],
                       key=lambda hd: (hd.layer_index, hd.is_final))
    weights = _resolve_weights(all_heads, options)
    wmap = {hd.key: w for hd, w in zip(all_heads, weights)}
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
    fwd_in = DistChannel(rank - 1, shape, act_dtype, dev) if s > 1 else None
    fwd_out = DistChannel(rank + 1, shape, act_dtype, dev) if s < P else None
    bwd_in = DistChannel(rank + 1, shape, act_dtype, dev) if s < P else None
    bwd_out = DistChannel(rank - 1, shape, act_dtype, dev) if s > 1 else None
    w = StageWorker(s, P, M, comp, data, fwd_in, fwd_out, bwd_in, bwd_out,
                    options.hoist_exit_heads)
    w.run()
    for ch in (fwd_out, bwd_out):
        if ch is not None:
            ch.flush()
    if w.exception is not None:
        raise w.exception
    grads = comp.tm.grads() if compute_factory is None else comp.grads()
    # tied replicas: all-reduce(sum) over the holders (every rank joins the
    # group creation; only holders take part in the reduction)
    for name, holders in sorted(part.tied_replicas.items()):
        group = dist.new_group([h - 1 for h in holders])
        if s in holders:
            g = grads[name]
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
    # this rank's view: its own stage's entries (event_log[s-1], memory[0])
    report = TrainStepReport(weights_used=tuple(weights), microbatches=M)
    report.event_log = [[] for _ in range(P)]
    report.event_log[s - 1] = list(w.event_log)
    report.memory = [StageMemoryCounters(s, w.max_in_flight)]
    report.wall_clock = {"forward": w.wall["F"], "backward": w.wall["B"],
                         "total": w.wall["F"] + w.wall["B"]}
    for key, vals in comp.head_losses.items():
        report.per_exit_losses[key] = sum(float(v) for v in vals) / len(vals)
    report.activation_messages[s] = fwd_out.count if fwd_out is not None else 0
    report.gradient_messages[s] = bwd_out.count if bwd_out is not None else 0
    return grads, report
