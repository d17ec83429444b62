"""Bubble filling: the plan / rescale algebra against the
reference's own KATs (tests/test_bubblefill.py:21-67 of eepipe), and the
threaded 1F1B executor with Part-1 / Part-2 fill microbatches against an
exact float64 gradient oracle of the filled objective, on CPU through the
executor's compute plug-in (the GPU restatement of the reference's executor
fill tests is tests/test_gpu_pipeline_suite.py).

Filled gradient (eepipe/pipeline.py:537-590, eepipe/bubblefill.py:96-121):
  sum over regular microbatches of sum_e w'_e CE_e
  + Part-1 fill i (depth d): sum over non-final exits on stages <= d of w'_e CE_e
  + Part-2 fill i (covered stages C): sum over heads on C of w'_e CE_e, with
    the gradient reaching only the parameters of C
  then each stage's gradient x grad_scale(stage);  w'_e = w_e x
  weight_scale(stage of e) for non-final exits.
"""
import numpy as np
import pytest
import torch

from paper_2312_04916_b200.bubblefill import (FillPlan, fill_rescale, has_rescale_overlap,
                                              part1_loss_sample_counts,
                                              part2_stage_sample_counts, plan_bubble_fill,
                                              truncated_part1_depths)
from paper_2312_04916_b200.errors import ConfigError
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition
from paper_2312_04916_b200.pipeline import IterationOptions, apply_fill, run_iteration_1f1b
from paper_2312_04916_b200 import schedule as sched

VOCAB = 32


# ---- plan / rescale algebra: the reference's KATs ---------------------------

def test_plan_capacity_formula_examples():
    plan = plan_bubble_fill(4, 0.5)
    assert plan.k_part1 == 2
    assert plan.part1_fwd_depths == (2, 1)
    assert plan.part2_bwd_depths == (2, 1)
    assert plan_bubble_fill(4, 3.0).empty
    assert plan_bubble_fill(8, 0.25).k_part1 == 5


def test_plan_rejects_bad_inputs():
    with pytest.raises(ConfigError):
        plan_bubble_fill(1, 0.5)
    with pytest.raises(ConfigError):
        plan_bubble_fill(4, 0.0)


def test_part1_truncation_to_deepest_exit_stage():
    plan = plan_bubble_fill(4, 0.5)
    assert truncated_part1_depths(plan, [2, 3]) == [2, None]
    assert truncated_part1_depths(plan, [1]) == [1, 1]
    assert truncated_part1_depths(plan, []) == [None, None]


def test_sample_counts_and_rescale():
    plan = plan_bubble_fill(4, 0.5)
    assert part1_loss_sample_counts(plan, [1, 2]) == {1: 2, 2: 1}
    assert part2_stage_sample_counts(plan) == {3: 1, 4: 2}
    rs = fill_rescale(plan, [1, 2], num_microbatches=4)
    assert rs.weight_scale_for(1) == pytest.approx(4 / 6)
    assert rs.weight_scale_for(2) == pytest.approx(4 / 5)
    assert rs.grad_scale_for(4) == pytest.approx(4 / 6)
    assert rs.grad_scale_for(1) == 1.0
    assert not has_rescale_overlap(plan, [1, 2])


def test_overlap_detection():
    plan = FillPlan(4, 0.5, 1, 1, (2,), (3,))
    assert has_rescale_overlap(plan, [2])
    assert not has_rescale_overlap(plan, [])


def test_fill_action_lists_are_deadlock_free_and_complete():
    """Every stage's list holds each regular microbatch once each way and the
    fills it takes part in; a dependency replay finishes (no deadlock)."""
    P, M = 4, 4
    depths, p2 = [2, 1], (2, 1)
    lists = {s: sched.fill_actions(P, M, s, depths, p2) for s in range(1, P + 1)}
    covered = [set(range(P - r + 1, P + 1)) for r in p2]

    def dep(kind, i, s):
        if kind == sched.FWD:
            return (kind, i, s - 1) if s > 1 else None
        if kind == sched.BWD:
            return (kind, i, s + 1) if s < P else (sched.FWD, i, s)
        if kind == sched.FILL1_FWD:
            return (kind, i, s - 1) if s > 1 else None
        if kind == sched.FILL1_BWD:
            return (kind, i, s + 1) if s < depths[i - 1] else (sched.FILL1_FWD, i, s)
        if kind == sched.FILL2_FWD:
            return (kind, i, s - 1) if s > 1 else None
        return (kind, i, s + 1) if s < P else (sched.FILL2_FWD, i, s)

    done, pos = set(), {s: 0 for s in lists}
    while any(pos[s] < len(lists[s]) for s in lists):
        moved = False
        for s in lists:
            while pos[s] < len(lists[s]):
                kind, i = lists[s][pos[s]]
                d = dep(kind, i, s)
                if d is not None and d not in done:
                    break
                done.add((kind, i, s))
                pos[s] += 1
                moved = True
        assert moved, "deadlock"
    for s in range(1, P + 1):
        acts = lists[s]
        assert sorted(i for k, i in acts if k == sched.FWD) == list(range(1, M + 1))
        assert sorted(i for k, i in acts if k == sched.BWD) == list(range(1, M + 1))
        assert sorted(i for k, i in acts if k == sched.FILL1_FWD) == \
            [i for i, d in enumerate(depths, 1) if d >= s]
        assert sorted(i for k, i in acts if k == sched.FILL2_FWD) == [1, 2]
        assert sorted(i for k, i in acts if k == sched.FILL2_BWD) == \
            [i for i, c in enumerate(covered, 1) if s in c]


# ---- executor on CPU: exact float64 against the filled-objective oracle ------

class FillToyCompute:
    """CPU float64 stage compute with the StageCompute fill interface:
    layer l: x <- x + tanh(x @ A_l); heads: mean CE of x @ out^T."""

    def __init__(self, spec, cfg, wmap, params):
        self.spec, self.cfg, self.weights = spec, cfg, wmap
        self.device = torch.device("cpu")
        self.act_dtype = torch.float64
        self.p = {n: params[n].clone().requires_grad_() for n in spec.params}
        self.head_losses = {hd.key: [] for _, hd in spec.heads}

    def forward(self, src, targets, grad=True):
        with torch.set_grad_enabled(grad):
            if self.spec.has_embedding:
                t = torch.as_tensor(np.asarray(src))
                x_in = None
                x = self.p["tok_emb"][t] + self.p["pos_emb"][torch.arange(t.shape[1])][None]
            else:
                x_in = src.detach().requires_grad_(grad)
                x = x_in
            taps = {0: x}
            for local, l in enumerate(self.spec.layer_indices, start=1):
                x = x + torch.tanh(x @ self.p[f"layer{l}.wq"])
                taps[local] = x
        return x, (x_in, x, taps, targets)

    def local_loss(self, st, include_final=True, record=True):
        _, _, taps, targets = st
        t = torch.as_tensor(np.asarray(targets)).reshape(-1)
        loss = None
        for local, hd in self.spec.heads:
            if hd.is_final and not include_final:
                continue
            xi = taps[local].reshape(-1, self.cfg.hidden_dim)
            lg = xi @ self.p[hd.param_names["out"]].t()
            ce = (torch.logsumexp(lg, -1) - lg[torch.arange(lg.shape[0]), t]).mean()
            if record:
                self.head_losses[hd.key].append(float(ce.detach()))
            term = ce * self.weights[hd.key]
            loss = term if loss is None else loss + term
        return loss

    def backward(self, st, g, loss=None, include_final=True, record=True):
        x_in, x_out, _, _ = st
        if loss is None:
            loss = self.local_loss(st, include_final, record)
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


def _setup(seed):
    cfg = ModelConfig(8, 16, 2, VOCAB, 12,
                      exits=(ExitSpec(2, loss_weight=0.3), ExitSpec(4, loss_weight=0.6)))
    model = build_model(cfg, seed)
    part = partition(model, 4)
    params = {n: torch.from_numpy(p.data.copy()) for n, p in model.params.items()}
    rng = np.random.default_rng(seed + 1)
    return model, part, params, rng


def _run(part, params, batch, plan=None, fill_rows=None, mb=2):
    factory = lambda spec, c, wmap: FillToyCompute(spec, c, wmap, params)  # noqa: E731
    g, rep = run_iteration_1f1b(part, batch, IterationOptions(
        microbatch_size=mb, fill_plan=plan, fill_batch=fill_rows), compute_factory=factory)
    return {n: t.detach().numpy() for n, t in g.items()}, rep


def _oracle(model, part, params, batch, plan, fill_rows, mb=2):
    """The filled objective's gradient, single process (module docstring)."""
    cfg = model.config
    p = {n: t.clone().requires_grad_() for n, t in params.items()}
    stage_of = {n: st.index for st in part.stages for n in st.params}
    M = batch.shape[0] // mb
    heads = sorted(model.heads, key=lambda hd: (hd.layer_index, hd.is_final))
    w = {hd.key: hd.loss_weight for hd in heads}
    depths, rescale = apply_fill(plan, part, M) if plan is not None else ([], None)
    if rescale is not None:
        for hd in heads:
            if not hd.is_final:
                w[hd.key] *= rescale.weight_scale_for(part.stage_of_head(hd.key))
    first_layer = {st.index: st.layer_indices[0] for st in part.stages}

    def objective(rows, head_ok, cut_stage=None):
        t_in, t_out = torch.as_tensor(rows[:, :-1]), torch.as_tensor(rows[:, 1:]).reshape(-1)
        # the fill's backward stops at the input of its deepest covered stage
        # (a head tapping that input belongs to the covered stage)
        cut_after = first_layer[cut_stage] - 1 if cut_stage is not None else None
        x = p["tok_emb"][t_in] + p["pos_emb"][torch.arange(t_in.shape[1])][None]
        if cut_after == 0:
            x = x.detach()
        taps = {0: x}
        for l in range(1, cfg.num_layers + 1):
            x = x + torch.tanh(x @ p[f"layer{l}.wq"])
            if l == cut_after:
                x = x.detach()
            taps[l] = x
        loss = 0.0
        for hd in heads:
            if head_ok(hd):
                xi = taps[hd.layer_index].reshape(-1, cfg.hidden_dim)
                lg = xi @ p[hd.param_names["out"]].t()
                loss = loss + w[hd.key] * (torch.logsumexp(lg, -1)
                                           - lg[torch.arange(lg.shape[0]), t_out]).mean()
        return loss

    total = 0.0
    for k in range(M):
        total = total + objective(batch[k * mb:(k + 1) * mb], lambda hd: True)
    k = 0
    if plan is not None:
        for d in depths:
            if d is None:
                continue
            rows = fill_rows[k * mb:(k + 1) * mb]
            k += 1
            total = total + objective(rows, lambda hd, d=d: not hd.is_final and
                                      part.stage_of_head(hd.key) <= d)
        for r in plan.part2_bwd_depths:
            rows = fill_rows[k * mb:(k + 1) * mb]
            k += 1
            deepest = part.num_stages - r + 1
            total = total + objective(rows, lambda hd, c=deepest: part.stage_of_head(hd.key) >= c,
                                      cut_stage=deepest)
    total.backward()
    out = {}
    for n, t in p.items():
        if t.grad is None:
            continue
        gs = rescale.grad_scale_for(stage_of[n]) if rescale is not None else 1.0
        out[n] = t.grad.numpy() * gs
    return out


def test_empty_plan_is_plain_1f1b():
    model, part, params, rng = _setup(19)
    batch = rng.integers(0, VOCAB, size=(8, 9))
    plain, _ = _run(part, params, batch)
    empty, _ = _run(part, params, batch, plan_bubble_fill(4, 3.0))
    for n in plain:
        assert np.array_equal(plain[n], empty[n])


def test_part2_gradient_touches_only_last_stages():
    """The reference's tests/test_pipeline.py:269-290 on the CPU compute."""
    model, part, params, rng = _setup(11)
    batch = rng.integers(0, VOCAB, size=(8, 9))
    fill_rows = rng.integers(0, VOCAB, size=(2, 9))
    plan = FillPlan(4, 0.5, 0, 1, (), (2,))
    plain, _ = _run(part, params, batch)
    filled, rep = _run(part, params, batch, plan, fill_rows)
    fill_only = _oracle(model, part, params, fill_rows, None, None)
    covered = {n for st in part.stages if st.index >= 3 for n in st.params}
    b = 4
    for n in plain:
        if n in covered:
            np.testing.assert_allclose(filled[n], (plain[n] + fill_only[n]) * (b / (b + 1)),
                                       rtol=1e-12, atol=1e-15)
        else:
            np.testing.assert_array_equal(filled[n], plain[n])
    assert rep.microbatches == 5


def test_part2_rescale_recovers_mean_over_extra_sample():
    """The reference's tests/test_pipeline.py:293-308: a full-depth Part-2
    insertion scaled by 4/5 equals the plain mean over all 5 microbatches."""
    model, part, params, rng = _setup(13)
    batch = rng.integers(0, VOCAB, size=(8, 9))
    fill_rows = rng.integers(0, VOCAB, size=(2, 9))
    filled, _ = _run(part, params, batch, FillPlan(4, 0.5, 0, 1, (), (4,)), fill_rows)
    all_rows = np.concatenate([batch, fill_rows], axis=0)
    every = _oracle(model, part, params, all_rows, None, None)
    for n in filled:
        np.testing.assert_allclose(filled[n] / 4.0, every[n] / 5.0, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("f_over_b,seed", [(0.5, 17), (0.25, 23)])
def test_full_fill_plan_matches_filled_objective(f_over_b, seed):
    """Part 1 (truncated to exit stages, final head excluded, loss weights
    rescaled) and Part 2 (suffix backward, stage gradients rescaled) together,
    exact in float64; losses are reported over the regular microbatches."""
    model, part, params, rng = _setup(seed)
    plan = plan_bubble_fill(4, f_over_b)
    depths, _ = apply_fill(plan, part, 4)
    n_extra = sum(1 for d in depths if d is not None) + plan.k_part2
    batch = rng.integers(0, VOCAB, size=(8, 9))
    fill_rows = rng.integers(0, VOCAB, size=(2 * n_extra, 9))
    filled, rep = _run(part, params, batch, plan, fill_rows)
    want = _oracle(model, part, params, batch, plan, fill_rows)
    assert set(filled) == set(want)
    for n in want:
        np.testing.assert_allclose(filled[n], want[n], rtol=1e-10, atol=1e-13)
    assert rep.microbatches == 4 + n_extra
    # every stage executed exactly the simulated timeline's order
    # (the first check of eepipe's verify_against_replay)
    for s in range(1, 5):
        assert rep.event_log[s - 1] == rep.timeline.order(s), s
    assert max(m.peak_fill_stored for m in rep.memory) >= 1


def test_fill_rejects_tied_parameters_and_bad_inputs():
    cfg = ModelConfig(4, 16, 2, VOCAB, 12, exits=(ExitSpec(1), ExitSpec(2)), tie_embeddings=True)
    with pytest.raises(ConfigError):
        apply_fill(plan_bubble_fill(4, 0.5), partition(build_model(cfg, 0), 4), 4)
    cfg = ModelConfig(4, 16, 2, VOCAB, 12, exits=(ExitSpec(1),))
    with pytest.raises(ConfigError):
        apply_fill(plan_bubble_fill(4, 0.5), partition(build_model(cfg, 0), 2), 4)
    model, part, params, rng = _setup(5)
    batch = rng.integers(0, VOCAB, size=(8, 9))
    with pytest.raises(ConfigError):  # no fill batch
        _run(part, params, batch, plan_bubble_fill(4, 0.5))


def test_simulator_matches_reference_timelines():
    """schedule.simulate (structural lists, earliest-start list scheduling,
    Part-2 gap packing) reproduces the reference simulator's per-stage event
    order, span, analytic decomposition and bubble flag over 300+ timelines
    (P 2-8, M P..2P, four exit placements, three variants, with and without
    bubble filling; tests/golden/make_schedule.py)."""
    import json
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(here, "schedule.json")) as f:
        gold = json.load(f)
    assert len(gold) > 300
    for g in gold:
        c = sched.CostModel(g["P"], g["M"], exit_counts=tuple(g["exit_counts"]),
                            embed_fwd_time=0.3, p2p_latency=0.05)
        plan = plan_bubble_fill(g["P"], g["f_over_b"]) if g["f_over_b"] else None
        t = sched.simulate(c, g["variant"], plan)
        for s in range(1, g["P"] + 1):
            assert t.order(s) == [tuple(a) for a in g["orders"][s - 1]], (g["P"], g["M"], s)
        assert t.span == pytest.approx(g["span"], abs=1e-9)
        assert t.decomposition == pytest.approx(g["decomposition"])
        assert t.bubble_assumption_violated == g["violated"]
