"""Pipeline-based early-exit inference across GPUs, one process per stage
(torchrun), over torch.distributed P2P (NCCL over NVLink on B200 boxes).

Semantics are those of `eepipe/inference.py:406-539` (and of the threaded
`inference.generate_pipeline`): stage s owns layers ((s-1)L/P, sL] and the
heads `exit_stage_index` puts on it; it processes messages strictly in
position order; heads are checked only for the decide row; the shallowest
firing exit (or the final head) emits the token exactly once, and the
message keeps flowing to the last stage to fill the KV of the deeper
layers while stage 1 already runs the next token.

Transport (`pipeline.Wire`, option (a) — NCCL has no
ANY_SOURCE):
  * stage s -> s+1: a fixed-size int64 header (rows, decide position,
    emitted flag, stop flag, positions) on the host control group (gloo: no
    device sync per header), then the hidden rows over NCCL (or host-staged
    gloo when the stage processes share one GPU).  The rows stay float32:
    the residual stream is float32 in every mode, which keeps this mode
    bitwise equal to KV recomputation (a bf16 boundary would round it), and
    at h = 7168 a row is 28 KB -- latency, not bandwidth;
  * every stage s >= 2 -> stage 1: one status per message
    (position, emitted-here, token, exit layer) on the control group; stage 1
    receives statuses in stage order until one says "emitted" and drains the
    later stages' statuses for that token before their next ones (FIFO per
    source);
  * per-token confidences are gathered to rank 0 at the end.
Sends are non-blocking (isend) so a stage never waits on its consumer.

The per-stage math is an `Engine` (inference.py) on the rank's GPU; a
`stage_factory` hook lets the CPU tests drive the protocol under gloo with a
deterministic stand-in (tests/test_pipeline_infer_dist.py).
"""

from __future__ import annotations

import time

import numpy as np

from .errors import ConfigError
from .inference import GenerationTrace, _check_context, default_stage_times
from .pipeline import Wire
from .schedule import inference_latency

_HDR_FIXED = 4  # rows, decide_pos, emitted, stop


def _torch():
    import torch
    return torch


class GpuStage:
    """The rank's stage on its GPU: the `Engine` of its layer span and heads."""

    def __init__(self, spec, cfg, threshold, dtype=None):
        torch = _torch()
        from .inference import _engine_for
        heads = [hd for _, hd in spec.heads]
        self.spec, self.cfg, self.thr = spec, cfg, threshold
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.eng = _engine_for(spec, spec.params, heads, cfg, spec.layer_indices,
                               spec.has_embedding, dtype, self.device)
        self.eng.kv.reset()
        self.heads_at = {}
        for local, hd in spec.heads:
            hi = next(i for i, e in enumerate(self.eng.heads) if e.desc.key == hd.key)
            self.heads_at.setdefault(local, []).append(hi)
        self.x_dtype = torch.float32

    def embed(self, tokens, positions):
        e = self.eng
        with _torch().cuda.stream(e.stream):
            e.embed_rows(tokens, positions, 0)
            return e.x[:len(tokens)].clone()

    def process(self, rows, positions, decide_pos):
        """Run this stage's taps and layers; returns (out rows, evaluations)
        with evaluations = [(head_key, tap, fired, token, conf)] in order."""
        torch = _torch()
        e = self.eng
        evals = []
        # the rows were received (or embedded) on the caller's current stream
        e.stream.wait_stream(torch.cuda.current_stream(e.device))
        with torch.cuda.stream(e.stream):
            n = len(positions)
            e._grow(n)
            e.x[:n].copy_(rows)
            e.refresh_stats(0, n)
            r = positions.index(decide_pos) if decide_pos in positions else None

            def check(local):
                if local not in self.heads_at or r is None:
                    return
                e.upload_ctrl(list(positions) + [r])
                for k, hi in enumerate(self.heads_at[local]):
                    e.eval_head(e.heads[hi], e.ctrl_ptr(n), 1, self.thr, k)
                e.fetch_results(len(self.heads_at[local]))
                for k, hi in enumerate(self.heads_at[local]):
                    hd = e.heads[hi].desc
                    evals.append((hd.key, hd.layer_index, bool(e.h_fire[k, 0]) or hd.is_final,
                                  int(e.h_tok[k, 0]), float(e.h_conf[k, 0])))

            e.upload_ctrl(list(positions))
            check(0)
            stops = sorted(k for k in self.heads_at if k >= 1)
            nloc = len(self.spec.layer_indices)
            if not stops or stops[-1] != nloc:
                stops.append(nloc)
            local = 1
            max_pos = max(positions)
            for stop in stops:
                if stop >= local:
                    e.upload_ctrl(list(positions))
                    # the prompt message (positions 0..t0-1) is the prefill
                    e.run_layers(local - 1, stop, n, [n] * (stop - local + 1), max_pos, 0,
                                 prefill=positions[0] == 0)
                    e.kv.mark_written(local - 1, stop, list(positions), max_pos)
                    check(stop)
                    local = stop + 1
            out = e.x[:n].clone()
            e.stream.synchronize()
        return out, evals

    def kv_complete(self, upto):
        return self.eng.kv.complete(upto)


def generate_pipeline_dist(part, prompt, threshold, max_new_tokens, stage_times=None, *,
                           dtype=None, stage_factory=None):
    """Distributed pipeline-based inference; every rank calls this (rank r =
    stage r+1).  Rank 0 returns the `GenerationTrace`, other ranks None."""
    torch = _torch()
    dist = torch.distributed
    rank, world = dist.get_rank(), dist.get_world_size()
    P = part.num_stages
    if P < 2:
        raise ConfigError("pipeline inference needs at least 2 stages")
    if world != P:
        raise ConfigError(f"{world} ranks for {P} stages")
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise ConfigError("prompt must be non-empty")
    if not 0.0 < threshold <= 1.0:
        raise ConfigError("threshold must lie in (0, 1]")
    cfg = part.config
    _check_context(cfg, len(prompt) + max_new_tokens)
    s = rank + 1
    spec = part.stages[rank]
    stage = (GpuStage(spec, cfg, threshold, dtype) if stage_factory is None
             else stage_factory(spec, cfg, threshold))
    dev = stage.device
    h = cfg.hidden_dim
    t0 = len(prompt)
    max_rows = max(t0, 1)
    hdr_len = _HDR_FIXED + max_rows
    conf_log = {}
    wire = Wire()

    def send_msg(rows, positions, decide, emitted, stop=False):
        hdr = [len(positions), decide, int(emitted), int(stop)] + list(positions)
        wire.send_ints(hdr + [0] * (hdr_len - len(hdr)), rank + 1)
        if not stop:
            wire.send(rows.to(stage.x_dtype), rank + 1)

    def recv_msg():
        hv = wire.recv_ints(hdr_len, rank - 1)
        n, decide, emitted, stop = hv[:4]
        if stop:
            return None
        positions = hv[_HDR_FIXED:_HDR_FIXED + n]
        rows = wire.recv((n, h), stage.x_dtype, dev, rank - 1)
        return rows, positions, decide, bool(emitted)

    def first_fire(evals, already):
        for key, tap, fired, tok, conf in evals:
            conf_log.setdefault(decide_of[0], {})[key] = conf
        if already:
            return None
        for key, tap, fired, tok, conf in evals:
            if fired:
                return tok, tap
        return None

    decide_of = [0]
    trace = GenerationTrace(prompt, threshold, "pipeline-dist") if rank == 0 else None

    if rank == 0:
        got = [0] * (P + 1)  # statuses received per stage (FIFO per source)
        t_start = time.perf_counter()
        t_last = t_start
        rows = stage.embed(prompt, list(range(t0)))
        positions, decide = list(range(t0)), t0 - 1
        position = t0 - 1
        for i in range(max_new_tokens):
            decide_of[0] = decide
            out, evals = stage.process(rows, positions, decide)
            emit = first_fire(evals, False)
            send_msg(out, positions, decide, emit is not None)
            msg_index = i  # the i-th message; every later stage answers it once
            if emit is not None:
                token, layer, estage = emit[0], emit[1], 1
            else:
                token = None
                for src in range(2, P + 1):
                    while got[src] <= msg_index:
                        pos, here, tok, lay = wire.recv_ints(4, src - 1)
                        got[src] += 1
                        if got[src] - 1 == msg_index and here and token is None:
                            token, layer, estage = tok, lay, src
                    if token is not None:
                        break
                if token is None:
                    raise ConfigError("no stage emitted a token")
            trace.tokens.append(int(token))
            trace.exit_layers.append(int(layer))
            trace.exit_stages.append(int(estage))
            now = time.perf_counter()
            trace.measured_latencies.append(now - t_last)
            t_last = now
            if i == max_new_tokens - 1:
                break
            position += 1
            rows = stage.embed([token], [position])
            positions, decide = [position], position
        send_msg(None, [], -1, True, stop=True)
        # drain the remaining statuses so every send is matched
        for src in range(2, P + 1):
            while got[src] < max_new_tokens:
                wire.recv_ints(4, src - 1)
                got[src] += 1
    else:
        while True:
            msg = recv_msg()
            if msg is None:
                if rank + 1 < world:
                    send_msg(None, [], -1, True, stop=True)
                break
            rows, positions, decide, emitted = msg
            decide_of[0] = decide
            out, evals = stage.process(rows, positions, decide)
            emit = first_fire(evals, emitted)
            here = emit is not None
            wire.send_ints([decide, int(here), emit[0] if here else -1,
                            emit[1] if here else -1], 0)
            if rank + 1 < world:
                send_msg(out, positions, decide, emitted or here)
    wire.flush()
    complete = stage.kv_complete(t0 + max_new_tokens - 1)
    logs = [None] * world
    dist.all_gather_object(logs, (conf_log, complete))
    if rank != 0:
        return None
    trace.measured_total = time.perf_counter() - t_start
    if not all(c for _, c in logs):
        raise ConfigError("KV fill mask incomplete after generation")
    merged = {}
    for cl, _ in logs:
        for pos, d in cl.items():
            merged.setdefault(pos, {}).update(d)
    gen = len(trace.tokens)
    trace.confidences = [merged.get(t0 - 1 + i, {}) for i in range(gen)]
    times = stage_times if stage_times is not None else default_stage_times(part)
    lat = inference_latency(trace.exit_stages, times)
    trace.latencies = lat["pipeline_per_token"]
    trace.total_latency = lat["pipeline_total"]
    trace.baseline_latency = lat["sequential_total"]
    return trace
