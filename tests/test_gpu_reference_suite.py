"""The reference's own behavioural tests (`pkg/tests/test_inference.py`,
`pkg/tests/test_model.py` of eepipe) restated against this package on the
GPU, same names / inputs / assertions.  Where the reference asserts bitwise
equality of training-forward results that depend on batched library matmuls
(batch permutation), the restatement uses a tight tolerance and says so."""
import numpy as np
import pytest

from paper_2312_04916_b200.errors import ConfigError, NonFiniteError, TokenError
from paper_2312_04916_b200.inference import (compare_modes, exit_decision, generate_kv_recompute,
                                             generate_pipeline, greedy_reference)
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

pytestmark = pytest.mark.gpu

VOCAB = 64
THR_FORCING_EXITS = 0.99 / VOCAB
THR_NO_EXITS = 6.0 / VOCAB


@pytest.fixture(scope="module")
def small_model():
    cfg = ModelConfig(8, 32, 4, VOCAB, 48,
                      exits=(ExitSpec(2, loss_weight=0.3), ExitSpec(4, loss_weight=0.6)))
    return build_model(cfg, 7)


@pytest.fixture(scope="module")
def small_part(small_model):
    return partition(small_model, 4)


def prompts_for(model, n, length=6):
    rng = np.random.default_rng(17)
    return [list(rng.integers(0, model.config.vocab_size, size=length)) for _ in range(n)]


# ---- tests/test_inference.py ------------------------------------------------------

def test_exit_decision_uniform():  # :47-51
    fire, token, conf = exit_decision(np.zeros(4), 0.25)
    assert conf == pytest.approx(0.25)
    assert not fire
    assert token == 0


def test_exit_decision_confident():  # :54-58
    logits = np.zeros(8)
    logits[3] = 30.0
    fire, token, conf = exit_decision(logits, 0.8)
    assert fire and token == 3 and conf > 0.999999


def test_exit_decision_threshold_one_never_fires():  # :61-65
    rng = np.random.default_rng(0)
    for _ in range(20):
        fire, _, _ = exit_decision(rng.normal(size=16) * 50, 1.0)
        assert not fire


def test_exit_decision_errors():  # :68-74
    with pytest.raises(NonFiniteError):
        exit_decision(np.array([np.inf, 0.0]), 0.5)
    with pytest.raises(ConfigError):
        exit_decision(np.zeros(4), 0.0)
    with pytest.raises(ConfigError):
        exit_decision(np.zeros(4), 1.5)


@pytest.mark.parametrize("threshold", [1.0, THR_NO_EXITS, THR_FORCING_EXITS])
@pytest.mark.parametrize("max_deferred", [1, 2, 4])
def test_modes_emit_identical_sequences(small_model, small_part, threshold, max_deferred):  # :106-114
    prompt = prompts_for(small_model, 1)[0]
    pipe = generate_pipeline(small_part, prompt, threshold, 12)
    reco = generate_kv_recompute(small_model, prompt, threshold, 12, max_deferred)
    assert pipe.tokens == reco.tokens
    assert pipe.exit_layers == reco.exit_layers
    assert pipe.confidences == reco.confidences


def test_forced_exits_actually_fire(small_model, small_part):  # :117-121
    pipe = generate_pipeline(small_part, prompts_for(small_model, 1)[0], THR_FORCING_EXITS, 12)
    assert any(e < small_model.config.num_layers for e in pipe.exit_layers)
    assert pipe.speedup > 1.0


def test_threshold_one_matches_uncached_greedy(small_model, small_part):  # :124-128
    for prompt in prompts_for(small_model, 2):
        ref = greedy_reference(small_model, prompt, 10)
        assert generate_pipeline(small_part, prompt, 1.0, 10).tokens == ref
        assert generate_kv_recompute(small_model, prompt, 1.0, 10).tokens == ref


def test_threshold_one_speedup_is_one(small_model, small_part):  # :131-134
    prompt = prompts_for(small_model, 1)[0]
    assert generate_pipeline(small_part, prompt, 1.0, 8).speedup == pytest.approx(1.0)
    assert generate_kv_recompute(small_model, prompt, 1.0, 8).speedup == pytest.approx(1.0)


def test_compare_modes_report(small_model, small_part):  # :150-156
    report = compare_modes(small_model, small_part, prompts_for(small_model, 3),
                           [1.0, THR_FORCING_EXITS], max_new_tokens=8)
    assert report["divergences"] == []
    assert len(report["runs"]) == 6
    base = [r for r in report["runs"] if r["threshold"] == 1.0]
    assert all(r["pipeline_speedup"] == pytest.approx(1.0) for r in base)


def test_mean_exit_depth_monotone_in_threshold(small_model, small_part):  # :159-168
    prompt = prompts_for(small_model, 1)[0]
    hi = generate_pipeline(small_part, prompt, THR_NO_EXITS, 12)
    lo = generate_pipeline(small_part, prompt, THR_FORCING_EXITS, 12)
    for t_hi, t_lo, e_hi, e_lo in zip(hi.tokens, lo.tokens, hi.exit_layers, lo.exit_layers):
        assert e_lo <= e_hi
        if t_hi != t_lo:
            break


def test_determinism(small_model, small_part):  # :171-178
    prompt = prompts_for(small_model, 1)[0]
    a = generate_pipeline(small_part, prompt, THR_FORCING_EXITS, 10)
    b = generate_pipeline(small_part, prompt, THR_FORCING_EXITS, 10)
    assert a.tokens == b.tokens and a.confidences == b.confidences
    c = generate_kv_recompute(small_model, prompt, THR_FORCING_EXITS, 10)
    d = generate_kv_recompute(small_model, prompt, THR_FORCING_EXITS, 10)
    assert c.tokens == d.tokens and c.confidences == d.confidences


def test_trace_records(small_model, small_part):  # :181-187
    prompt = prompts_for(small_model, 1)[0]
    tr = generate_pipeline(small_part, prompt, 1.0, 5)
    recs = list(tr.records())
    assert len(recs) == 5
    assert recs[0]["position"] == len(prompt)
    assert set(recs[0]["confidence"]) == {"exit_l2", "exit_l4", "final"}


def test_pipeline_needs_two_stages(small_model):  # :195-198
    with pytest.raises(ConfigError):
        generate_pipeline(partition(small_model, 1), [1, 2, 3], 1.0, 4)


def test_context_overflow(small_model, small_part):  # :201-206
    long_prompt = [0] * small_model.config.max_seq_len
    with pytest.raises(TokenError):
        generate_kv_recompute(small_model, long_prompt, 1.0, 4)
    with pytest.raises(TokenError):
        generate_pipeline(small_part, long_prompt, 1.0, 4)


def test_mlp_head_supported_in_inference():  # :226-233
    cfg = ModelConfig(4, 32, 4, VOCAB, 32, exits=(ExitSpec(2, "mlp+embed", 0.5),))
    model = build_model(cfg, 0)
    part = partition(model, 2)
    prompt = [3, 1, 4]
    assert (generate_kv_recompute(model, prompt, 1.0, 6).tokens
            == generate_pipeline(part, prompt, 1.0, 6).tokens
            == greedy_reference(model, prompt, 6))


# ---- tests/test_model.py (training forward on the GPU) ----------------------------

def _small(**kw):
    base = dict(num_layers=4, hidden_dim=16, num_heads=2, vocab_size=32, max_seq_len=12)
    base.update(kw)
    return ModelConfig(**base)


def _tm(model):
    import torch
    from paper_2312_04916_b200.training import TrainModel
    return TrainModel(model, dtype=torch.float32)


def test_exits_are_readonly_taps():  # test_model.py:62-71
    from paper_2312_04916_b200.training import forward_all_exits
    rng = np.random.default_rng(5)
    toks = rng.integers(0, 32, size=(2, 6))
    with_exits = forward_all_exits(_tm(build_model(_small(exits=(ExitSpec(1), ExitSpec(3))), 42)),
                                   toks)
    plain = forward_all_exits(_tm(build_model(_small(), 42)), toks)
    assert np.array_equal(with_exits[-1].detach().cpu().numpy(), plain[-1].detach().cpu().numpy())
    assert len(with_exits) == 3


def test_causality_at_every_exit():  # test_model.py:74-85
    from paper_2312_04916_b200.training import forward_all_exits
    rng = np.random.default_rng(6)
    model = _tm(build_model(_small(exits=(ExitSpec(0), ExitSpec(2))), 3))
    toks = rng.integers(0, 32, size=(1, 8))
    base = [o.detach().cpu().numpy() for o in forward_all_exits(model, toks)]
    t = 4
    perturbed = toks.copy()
    perturbed[0, t] = (perturbed[0, t] + 1) % 32
    for b, o in zip(base, forward_all_exits(model, perturbed)):
        o = o.detach().cpu().numpy()
        assert np.array_equal(b[:, :t, :], o[:, :t, :])
        assert not np.array_equal(b[:, t:, :], o[:, t:, :])


def test_batch_permutation_permutes_logits():  # test_model.py:88-95 (tolerance, see module doc)
    from paper_2312_04916_b200.training import forward_all_exits
    rng = np.random.default_rng(7)
    model = _tm(build_model(_small(exits=(ExitSpec(2),)), 9))
    toks = rng.integers(0, 32, size=(4, 6))
    perm = np.array([2, 0, 3, 1])
    for a, b in zip(forward_all_exits(model, toks), forward_all_exits(model, toks[perm])):
        np.testing.assert_allclose(a.detach().cpu().numpy()[perm], b.detach().cpu().numpy(),
                                   rtol=1e-5, atol=1e-6)


def test_weighted_loss_matches_hand_sum():  # test_model.py:98-107
    from paper_2312_04916_b200.training import weighted_loss
    rng = np.random.default_rng(8)
    model = _tm(build_model(_small(exits=(ExitSpec(1), ExitSpec(2))), 11))
    batch = rng.integers(0, 32, size=(2, 7))
    weights = [0.25, 0.5, 1.0]
    total, per_exit = weighted_loss(model, batch, weights)
    assert float(total.detach()) == pytest.approx(sum(w * l for w, l in zip(weights, per_exit)),
                                                  rel=1e-6)


def test_zero_weights_reduce_to_standard_loss():  # test_model.py:110-116
    from paper_2312_04916_b200.training import weighted_loss
    rng = np.random.default_rng(9)
    batch = rng.integers(0, 32, size=(2, 7))
    total, _ = weighted_loss(_tm(build_model(_small(exits=(ExitSpec(1), ExitSpec(2))), 4)), batch,
                             [0.0, 0.0, 1.0])
    plain, _ = weighted_loss(_tm(build_model(_small(), 4)), batch, [1.0])
    assert float(total.detach()) == pytest.approx(float(plain.detach()), rel=1e-6)


def test_weight_length_mismatch():  # test_model.py:119-122
    from paper_2312_04916_b200.training import weighted_loss
    with pytest.raises(Exception):
        weighted_loss(_tm(build_model(_small(exits=(ExitSpec(1),)), 0)), np.zeros((1, 4), dtype=int),
                      [1.0])


def test_overlong_sequence_rejected():  # test_model.py:125-129
    from paper_2312_04916_b200.training import forward_all_exits
    with pytest.raises(TokenError):
        forward_all_exits(_tm(build_model(_small(), 0)), np.zeros((1, 13), dtype=int))


def test_tied_gradient_equals_sum_of_untied_uses():  # test_model.py:132-156
    import torch
    from paper_2312_04916_b200.training import weighted_loss
    rng = np.random.default_rng(10)
    tied = _tm(build_model(_small(exits=(ExitSpec(1), ExitSpec(3)), tie_embeddings=True), 21))
    batch = rng.integers(0, 32, size=(2, 6))
    weights = [0.5, 0.5, 1.0]
    loss, _ = weighted_loss(tied, batch, weights)
    loss.backward()
    g_tied = tied.params["tok_emb"].grad.double().cpu().numpy()
    um = build_model(_small(exits=(ExitSpec(1), ExitSpec(3))), 21)
    shared = build_model(_small(exits=(ExitSpec(1), ExitSpec(3)), tie_embeddings=True),
                         21).params["tok_emb"].data
    for name in ("tok_emb", "exit_l1.out", "exit_l3.out"):
        um.params[name].data[...] = shared
    untied = _tm(um)
    loss, _ = weighted_loss(untied, batch, weights)
    loss.backward()
    g_sum = sum(untied.params[n].grad.double().cpu().numpy()
                for n in ("tok_emb", "exit_l1.out", "exit_l3.out"))
    np.testing.assert_allclose(g_tied, g_sum, rtol=1e-4, atol=1e-6)
