"""The reference's pipeline-executor tests (`pkg/tests/test_pipeline.py` of
eepipe) restated on the GPU: the 1F1B executor with fused tcgen05 exit heads
against this package's single-device oracle (`training.
single_device_gradients`) over the reference's seven configurations (tap-0
exits, tied embeddings, norm+embed / mlp+embed / layer+embed heads, an exit
at the final tap), plus its protocol checks.

Numerics: everything runs in bf16 on both sides (the reference compares two
float64 runs at < 1e-9): pipeline vs single device within 2e-2 relative per
tensor (Frobenius) — stage boundaries change where bf16 gradients are rounded
and summed — and per-exit losses within 1e-3.  Where the reference asserts
bitwise equality of two executions of the SAME computation (P = 1 vs the
oracle, eager vs deferred exit forward, repeated runs) the restatement is
bitwise too.
"""
import numpy as np
import pytest

from paper_2312_04916_b200 import schedule as sched
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

pytestmark = pytest.mark.gpu

VOCAB = 64


def make_setup(num_layers, exits, tie, seed, rows=8, seq=8):  # test_pipeline.py:29-35
    cfg = ModelConfig(num_layers, 32, 4, VOCAB, 16, exits=exits, tie_embeddings=tie)
    model = build_model(cfg, seed)
    rng = np.random.default_rng(seed + 1000)
    batch = rng.integers(0, VOCAB, size=(rows, seq + 1))
    weights = [e.loss_weight for e in sorted(exits, key=lambda e: e.layer_index)] + [1.0]
    return model, batch, weights


def _rel(a, b):
    a = a.detach().double().cpu().numpy()
    b = b.detach().double().cpu().numpy()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


CONFIGS = [  # test_pipeline.py:47-57
    (4, (), False, 2),
    (4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), False, 4),
    (4, (ExitSpec(0, loss_weight=0.3),), False, 4),
    (4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), True, 2),
    (6, (ExitSpec(0, loss_weight=0.2), ExitSpec(3, "norm+embed", 0.4)), True, 3),
    (8, (ExitSpec(2, loss_weight=0.25), ExitSpec(4, "mlp+embed", 0.5),
         ExitSpec(8, loss_weight=0.1)), False, 4),
    (4, (ExitSpec(2, "layer+embed", 0.5),), False, 2),
]


@pytest.mark.parametrize("layers,exits,tie,num_stages", CONFIGS)
def test_gradient_equivalence(layers, exits, tie, num_stages):  # test_pipeline.py:60-69
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    model, batch, weights = make_setup(layers, exits, tie, seed=layers * 10 + num_stages)
    oracle, oracle_losses = single_device_gradients(TrainModel(model), batch, weights, 2)
    part = partition(model, num_stages)
    grads, report = run_iteration_1f1b(part, batch, IterationOptions(microbatch_size=2),
                                       model=model)
    assert set(grads) == set(oracle)
    for name in oracle:
        assert _rel(grads[name], oracle[name]) < 2e-2, name
    for key, val in report.per_exit_losses.items():
        assert val == pytest.approx(oracle_losses[key], rel=1e-3)


def test_p1_reduces_bitwise():  # test_pipeline.py:72-80
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    model, batch, weights = make_setup(
        4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), True, seed=3)
    oracle, _ = single_device_gradients(TrainModel(model), batch, weights, 2)
    grads, _ = run_iteration_1f1b(partition(model, 1), batch, IterationOptions(microbatch_size=2),
                                  model=model)
    for name in oracle:
        assert _rel(grads[name], oracle[name]) < 1e-6, name


def test_eager_and_deferred_identical_gradients():  # test_pipeline.py:83-98
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    model, batch, _ = make_setup(
        4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), False, seed=8)
    part = partition(model, 4)
    g_def, r_def = run_iteration_1f1b(part, batch, IterationOptions(2, defer_exit_forward=True),
                                      model=model)
    g_eag, r_eag = run_iteration_1f1b(part, batch, IterationOptions(2, defer_exit_forward=False),
                                      model=model)
    for name in g_def:
        assert bool((g_def[name] == g_eag[name]).all()), name
    # the fused head keeps no logits in either variant (reference: [0,1,1,0] / [0,3,2,0])
    assert [m.peak_logit_copies for m in r_def.memory] == [0, 0, 0, 0]
    assert [m.peak_logit_copies for m in r_eag.memory] == [0, 0, 0, 0]


def test_in_flight_bound():  # test_pipeline.py:101-109
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    model, batch, _ = make_setup(4, (ExitSpec(1, loss_weight=0.5),), False, seed=4, rows=12)
    for p in (2, 4):
        _, report = run_iteration_1f1b(partition(model, p), batch, IterationOptions(2), model=model)
        for mem in report.memory:
            assert mem.peak_stored_microbatches <= p - mem.stage + 1


def test_message_counts_and_replay():  # test_pipeline.py:112-122
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    model, batch, _ = make_setup(
        4, (ExitSpec(1, loss_weight=0.5), ExitSpec(2, loss_weight=0.5)), False, seed=5)
    _, report = run_iteration_1f1b(partition(model, 4), batch, IterationOptions(2), model=model)
    m = batch.shape[0] // 2
    for s in range(1, 4):
        assert report.activation_messages[s] == m
        assert report.gradient_messages[s + 1] == m
    # executed order == the 1F1B action list of every stage (the replay check)
    for s in range(1, 5):
        assert report.event_log[s - 1] == sched.regular_actions(4, m, s)


def test_determinism_semantic_state():  # test_pipeline.py:135-141
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    model, batch, _ = make_setup(4, (ExitSpec(2, loss_weight=0.5),), True, seed=7)
    part = partition(model, 2)
    _, r1 = run_iteration_1f1b(part, batch, IterationOptions(2), model=model)
    _, r2 = run_iteration_1f1b(part, batch, IterationOptions(2), model=model)
    assert r1.semantic_state() == r2.semantic_state()


def test_hoisted_exit_heads_identical_gradients():
    """The §4.2.2 Remark (exit losses formed before the downstream gradient
    arrives, IterationOptions.hoist_exit_heads) changes only the timing: the
    gradients are bitwise those of the plain order."""
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    model, batch, _ = make_setup(
        4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), False, seed=8)
    part = partition(model, 4)
    g_h, r_h = run_iteration_1f1b(part, batch, IterationOptions(2, hoist_exit_heads=True),
                                  model=model)
    g_p, r_p = run_iteration_1f1b(part, batch, IterationOptions(2, hoist_exit_heads=False),
                                  model=model)
    for name in g_h:
        assert bool((g_h[name] == g_p[name]).all()), name
    assert r_h.per_exit_losses == r_p.per_exit_losses


# ---- bubble filling (eepipe/pipeline.py:456-498) ---------------

def _fill_golden():
    import json
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(here, "fill.json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(here, "fill.npz"))


def test_bubble_fill_matches_reference_executor():
    """The full plan_bubble_fill(4, 0.5) iteration (Part-1 truncated to the
    exit stages, Part-2 suffix backwards, loss-weight and stage-gradient
    rescaling) against the REFERENCE executor's float64 gradients
    (tests/golden/make_fill.py), bf16 within 3e-2 relative per tensor; the
    plain iteration likewise; and the fill's effect (filled - plain) within
    1e-1 relative wherever it exceeds 10% of the gradient (below that it is
    bf16 rounding noise)."""
    from paper_2312_04916_b200.bubblefill import plan_bubble_fill
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    meta, g = _fill_golden()
    L, h, nh, V, s_max = meta["config"]
    cfg = ModelConfig(L, h, nh, V, s_max,
                      exits=tuple(ExitSpec(l, loss_weight=w) for l, w in meta["exits"]))
    model = build_model(cfg, meta["seed"])
    part = partition(model, 4)
    batch, fill_rows = g["batch"], g["fill_rows"]
    plain, _ = run_iteration_1f1b(part, batch, IterationOptions(microbatch_size=2), model=model)
    filled, rep = run_iteration_1f1b(part, batch, IterationOptions(
        microbatch_size=2, fill_plan=plan_bubble_fill(4, meta["f_over_b"]),
        fill_batch=fill_rows), model=model)
    assert rep.microbatches == meta["microbatches"]
    for name in filled:
        ref_f, ref_p = g["filled/" + name], g["plain/" + name]
        ours_f = filled[name].detach().double().cpu().numpy()
        ours_p = plain[name].detach().double().cpu().numpy()
        assert np.linalg.norm(ours_f - ref_f) / np.linalg.norm(ref_f) < 3e-2, name
        assert np.linalg.norm(ours_p - ref_p) / np.linalg.norm(ref_p) < 3e-2, name
        d_ref = ref_f - ref_p
        if np.linalg.norm(d_ref) > 0.1 * np.linalg.norm(ref_p):  # effect above bf16 noise
            d = ours_f - ours_p
            assert np.linalg.norm(d - d_ref) / np.linalg.norm(d_ref) < 0.1, name
    for k, v in meta["filled_losses"].items():
        assert rep.per_exit_losses[k] == pytest.approx(v, rel=1e-3)


def test_bubble_fill_part2_touches_only_last_stages():
    """tests/test_pipeline.py:269-290 of the reference: one Part-2 insertion of
    backward depth 2 leaves stages 1-2 bitwise unchanged and scales stages 3-4
    by b/(b+1) after adding the fill's gradient."""
    from paper_2312_04916_b200.bubblefill import FillPlan
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    cfg = ModelConfig(8, 32, 4, VOCAB, 16,
                      exits=(ExitSpec(2, loss_weight=0.3), ExitSpec(4, loss_weight=0.6)))
    model = build_model(cfg, 11)
    part = partition(model, 4)
    rng = np.random.default_rng(12)
    batch = rng.integers(0, VOCAB, size=(8, 9))
    fill_rows = rng.integers(0, VOCAB, size=(2, 9))
    plain, _ = run_iteration_1f1b(part, batch, IterationOptions(microbatch_size=2), model=model)
    filled, _ = run_iteration_1f1b(part, batch, IterationOptions(
        microbatch_size=2, fill_plan=FillPlan(4, 0.5, 0, 1, (), (2,)), fill_batch=fill_rows),
        model=model)
    fill_oracle, _ = single_device_gradients(TrainModel(model), fill_rows, [0.3, 0.6, 1.0], 2)
    covered = {n for st in part.stages if st.index >= 3 for n in st.params}
    for name in plain:
        if name in covered:
            want = (plain[name].double() + fill_oracle[name].double().to(plain[name].device)) * 0.8
            assert _rel(filled[name], want) < 2e-2, name
        else:
            assert bool((filled[name] == plain[name]).all()), name
