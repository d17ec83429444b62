"""Pipeline host logic on CPU: 1F1B action lists, the ordered channel
protocol, and the distributed stage executor over torch.distributed (gloo,
world sizes 2 and 4) with a small CPU stage compute standing in for the GPU
one (the executor, channels and tied-replica all-reduce are the product code;
only the per-stage math is replaced).

Mirrors the reference's pipeline tests: in-flight bound P-s+1
(tests/test_pipeline.py:101-109), message counts (:112-122), queue protocol
(:356-372) and gradient equivalence with single-device training (:59-69).
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_04916_b200 import schedule as sched
from paper_2312_04916_b200.errors import QueueProtocolError
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition
from paper_2312_04916_b200.pipeline import (GradientMessage, IterationOptions, TaggedChannel,
                                            WeightSchedule, run_stage_1f1b_dist, weight_at_step)


def test_regular_actions_structure():
    for P in (1, 2, 4):
        for M in (1, 3, 8):
            for s in range(1, P + 1):
                acts = sched.regular_actions(P, M, s)
                assert sorted(k for kind, k in acts if kind == "F") == list(range(1, M + 1))
                assert sorted(k for kind, k in acts if kind == "B") == list(range(1, M + 1))
                assert sched.max_in_flight(acts) == min(P - s + 1, M)
                # a microbatch's backward follows its forward
                seen = set()
                for kind, k in acts:
                    if kind == "F":
                        seen.add(k)
                    else:
                        assert k in seen


def test_tagged_queue_rejects_out_of_order_regular_ids():
    """The reference's queue-protocol tests (tests/test_pipeline.py:354-372)."""
    q = TaggedChannel("t")
    q.send(GradientMessage(("mb", 2), None))
    q.send(GradientMessage(("mb", 1), None))
    q.recv(("mb", 2))
    with pytest.raises(QueueProtocolError):
        q.recv(("mb", 1))


def test_tagged_queue_stashes_fills():
    q = TaggedChannel("t")
    q.send(GradientMessage(("mb", 1), None))
    q.send(GradientMessage(("p1", 1), "fill"))
    q.send(GradientMessage(("mb", 2), None))
    assert q.recv(("p1", 1)).data == "fill"
    assert q.recv(("mb", 1)).mb == ("mb", 1)
    assert q.recv(2).mb == ("mb", 2)  # a bare int is a regular id


def test_weight_schedule():
    ws = WeightSchedule("linear", early=(0.0, 0.2), early_end=(1.0, 0.4), span_steps=10)
    assert weight_at_step(ws, 0) == [0.0, 0.2, 1.0]
    assert weight_at_step(ws, 5) == pytest.approx([0.5, 0.3, 1.0])
    assert weight_at_step(ws, 50) == pytest.approx([1.0, 0.4, 1.0])


# ---- a CPU stage compute with the StageCompute interface ---------------------

class ToyCompute:
    """Layer l: x <- x + tanh(x @ A_l); head: mean((x @ out^T)[.., t])-style
    loss = mean over rows of logsumexp(x W^T) - (x W^T)[t] (a real CE)."""

    def __init__(self, spec, cfg, wmap, params):
        self.spec, self.cfg, self.weights = spec, cfg, wmap
        self.device = torch.device("cpu")
        self.act_dtype = torch.float64
        self.p = {n: params[n].clone().requires_grad_() for n in spec.params}
        self.head_losses = {hd.key: [] for _, hd in spec.heads}

    def forward(self, src, targets):
        if self.spec.has_embedding:
            t = torch.as_tensor(np.asarray(src))
            x_in = None
            x = self.p["tok_emb"][t] + self.p["pos_emb"][torch.arange(t.shape[1])][None]
        else:
            x_in = src.detach().requires_grad_()
            x = x_in
        taps = {0: x}
        for local, l in enumerate(self.spec.layer_indices, start=1):
            x = x + torch.tanh(x @ self.p[f"layer{l}.wq"])
            taps[local] = x
        return x, (x_in, x, taps, targets)

    def backward(self, st, g):
        x_in, x_out, taps, targets = st
        loss = None
        t = torch.as_tensor(np.asarray(targets)).reshape(-1)
        for local, hd in self.spec.heads:
            xi = taps[local].reshape(-1, self.cfg.hidden_dim)
            lg = xi @ self.p[hd.param_names["out"]].t()
            ce = (torch.logsumexp(lg, -1) - lg[torch.arange(lg.shape[0]), t]).mean()
            self.head_losses[hd.key].append(float(ce))
            term = ce * self.weights[hd.key]
            loss = term if loss is None else loss + term
        outs, grads = [], []
        if loss is not None:
            outs.append(loss)
            grads.append(torch.ones_like(loss))
        if g is not None:
            outs.append(x_out)
            grads.append(g)
        torch.autograd.backward(outs, grads)
        return None if x_in is None else x_in.grad

    def grads(self):
        return {n: p.grad for n, p in self.p.items() if p.grad is not None}


def _toy_reference(model, batch, weights, mb):
    """Single-process, same microbatching, same math: gradient oracle."""
    p = {n: torch.from_numpy(a.data.copy()).requires_grad_() for n, a in model.params.items()}
    cfg = model.config
    for k in range(batch.shape[0] // mb):
        rows = batch[k * mb:(k + 1) * mb]
        t_in, t_out = torch.as_tensor(rows[:, :-1]), torch.as_tensor(rows[:, 1:]).reshape(-1)
        x = p["tok_emb"][t_in] + p["pos_emb"][torch.arange(t_in.shape[1])][None]
        taps = {0: x}
        for l in range(1, cfg.num_layers + 1):
            x = x + torch.tanh(x @ p[f"layer{l}.wq"])
            taps[l] = x
        loss = 0.0
        for hd, w in zip(model.heads, weights):
            xi = taps[hd.layer_index].reshape(-1, cfg.hidden_dim)
            lg = xi @ p[hd.param_names["out"]].t()
            loss = loss + w * (torch.logsumexp(lg, -1) - lg[torch.arange(lg.shape[0]), t_out]).mean()
        loss.backward()
    return {n: t.grad for n, t in p.items() if t.grad is not None}


def _worker(rank, world, port, cfg_args, tied, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = ModelConfig(*cfg_args[:5], exits=cfg_args[5], tie_embeddings=tied)
        model = build_model(cfg, 3)
        part = partition(model, world)
        batch = np.random.default_rng(9).integers(0, cfg.vocab_size, size=(8, 9))
        params = {n: torch.from_numpy(p.data.copy()) for n, p in model.params.items()}
        factory = lambda spec, c, wmap: ToyCompute(spec, c, wmap, params)  # noqa: E731
        grads, rep = run_stage_1f1b_dist(part, batch, IterationOptions(microbatch_size=2),
                                         compute_factory=factory)
        q.put((rank, {n: g.numpy() for n, g in grads.items()}, rep.event_log,
               rep.max_in_flight, rep.activation_messages, rep.gradient_messages))
    except BaseException as exc:  # pragma: no cover - reported by the parent
        q.put((rank, repr(exc), None, None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tied", [(2, False), (4, False), (2, True), (4, True)])
def test_distributed_1f1b_matches_single_process(world, tied):
    exits = (ExitSpec(1, loss_weight=0.3), ExitSpec(2, loss_weight=0.6))
    cfg_args = (4, 16, 2, 32, 12, exits)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + np.random.default_rng().integers(0, 2000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_args, tied, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in results:
        assert not isinstance(r[1], str), r[1]
    cfg = ModelConfig(*cfg_args[:5], exits=exits, tie_embeddings=tied)
    model = build_model(cfg, 3)
    batch = np.random.default_rng(9).integers(0, cfg.vocab_size, size=(8, 9))
    ref = _toy_reference(model, batch, [hd.loss_weight for hd in model.heads], 2)
    merged = {}
    for rank, grads, log, inflight, acts, gms in sorted(results, key=lambda r: r[0]):
        s = rank + 1
        assert log[s - 1] == sched.regular_actions(world, 4, s)
        assert inflight[s] == min(world - s + 1, 4)
        if s < world:
            assert acts[s] == 4
        if s > 1:
            assert gms[s] == 4
        for n, g in grads.items():
            if n in merged:  # tied replicas: all-reduced, so every holder agrees
                np.testing.assert_allclose(merged[n], g, rtol=1e-12, atol=1e-15)
            merged[n] = g
    assert set(merged) == set(ref)
    for n in ref:
        np.testing.assert_allclose(merged[n], ref[n].numpy(), rtol=1e-9, atol=1e-12)


def _fill_worker(rank, world, port, q):
    """One rank of a distributed iteration WITH bubble filling (gloo, CPU
    float64 compute): fill traffic travels over the tagged point-to-point
    channel (headers carry (kind, index); early arrivals are stashed)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from test_bubblefill import FillToyCompute, _setup
        from paper_2312_04916_b200.bubblefill import plan_bubble_fill
        from paper_2312_04916_b200.pipeline import apply_fill
        model, part, params, rng = _setup(17)
        plan = plan_bubble_fill(4, 0.5)
        depths, _ = apply_fill(plan, part, 4)
        n_extra = sum(1 for d in depths if d is not None) + plan.k_part2
        batch = rng.integers(0, 32, size=(8, 9))
        fill_rows = rng.integers(0, 32, size=(2 * n_extra, 9))
        factory = lambda spec, c, wmap: FillToyCompute(spec, c, wmap, params)  # noqa: E731
        grads, rep = run_stage_1f1b_dist(
            part, batch, IterationOptions(microbatch_size=2, fill_plan=plan,
                                          fill_batch=fill_rows),
            compute_factory=factory)
        q.put((rank, {n: g.detach().numpy() for n, g in grads.items()}, rep.event_log,
               [list(o) for o in (rep.timeline.order(s) for s in range(1, 5))],
               rep.microbatches))
    except BaseException as exc:  # pragma: no cover - reported by the parent
        q.put((rank, repr(exc), None, None, None))
    finally:
        dist.destroy_process_group()


def test_distributed_bubble_fill_matches_threaded_executor():
    """Bubble filling over torch.distributed (4 ranks, gloo): every rank runs
    the simulated timeline's order, the fill microbatches travel as tagged
    messages, and the merged gradients equal the single-process threaded
    executor's bitwise (float64, same per-stage accumulation order)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_bubblefill import FillToyCompute, _setup
    from paper_2312_04916_b200.bubblefill import plan_bubble_fill
    from paper_2312_04916_b200.pipeline import apply_fill, run_iteration_1f1b
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + np.random.default_rng().integers(2000, 4000)
    procs = [ctx.Process(target=_fill_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
    for r in results:
        assert not isinstance(r[1], str), r[1]
    model, part, params, rng = _setup(17)
    plan = plan_bubble_fill(4, 0.5)
    depths, _ = apply_fill(plan, part, 4)
    n_extra = sum(1 for d in depths if d is not None) + plan.k_part2
    batch = rng.integers(0, 32, size=(8, 9))
    fill_rows = rng.integers(0, 32, size=(2 * n_extra, 9))
    factory = lambda spec, c, wmap: FillToyCompute(spec, c, wmap, params)  # noqa: E731
    ref, rep_ref = run_iteration_1f1b(part, batch, IterationOptions(
        microbatch_size=2, fill_plan=plan, fill_batch=fill_rows), compute_factory=factory)
    merged = {}
    for rank, grads, log, orders, nmb in sorted(results, key=lambda r: r[0]):
        s = rank + 1
        assert log[s - 1] == [tuple(a) for a in orders[s - 1]]
        assert nmb == rep_ref.microbatches
        merged.update(grads)
    assert set(merged) == set(ref)
    for n in ref:
        assert np.array_equal(merged[n], ref[n].detach().numpy()), n
