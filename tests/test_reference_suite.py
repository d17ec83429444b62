"""The reference's own structural tests (`pkg/tests/test_model.py`,
`pkg/tests/test_inference.py` of eepipe), restated against this package's API
with the same names, inputs and assertions: a caller's existing test suite
reads the same here.  CPU-only items (configuration, partition, checkpoint,
KV-cache discipline); the GPU items are in tests/test_gpu_reference_suite.py.
"""
import numpy as np
import pytest

from paper_2312_04916_b200.checkpoint import load_model, save_model
from paper_2312_04916_b200.errors import ConfigError
from paper_2312_04916_b200.inference import KVCache
from paper_2312_04916_b200.model import (ExitSpec, ModelConfig, build_model, exit_stage_index,
                                         expected_param_count, partition)


def small_config(**kw):
    base = dict(num_layers=4, hidden_dim=16, num_heads=2, vocab_size=32, max_seq_len=12)
    base.update(kw)
    return ModelConfig(**base)


# ---- tests/test_model.py -------------------------------------------------------

def test_param_count_matches_enumeration():  # test_model.py:31-40
    for exits, tie in [
        ((), False),
        ((ExitSpec(2), ExitSpec(4)), False),
        ((ExitSpec(0), ExitSpec(1, "norm+embed"), ExitSpec(3, "mlp+embed")), True),
        ((ExitSpec(2, "layer+embed"),), False),
    ]:
        cfg = small_config(exits=exits, tie_embeddings=tie)
        model = build_model(cfg, 7)
        assert model.param_count() == expected_param_count(cfg)


def test_tied_saves_one_matrix_per_exit():  # test_model.py:43-48
    exits = (ExitSpec(1), ExitSpec(3))
    untied = build_model(small_config(exits=exits), 0)
    tied = build_model(small_config(exits=exits, tie_embeddings=True), 0)
    assert untied.param_count() - tied.param_count() == 2 * 32 * 16


def test_head_count_and_order():  # test_model.py:51-59 (structure part)
    model = build_model(small_config(exits=(ExitSpec(2), ExitSpec(1))), 1)
    assert [h.layer_index for h in model.heads] == [1, 2, 4]
    assert model.heads[-1].is_final
    assert len(build_model(small_config(), 1).heads) == 1


def test_exit_stage_rule():  # test_model.py:159-165
    assert exit_stage_index(2, 8, 4) == 2
    assert exit_stage_index(4, 8, 4) == 3
    assert exit_stage_index(0, 8, 4) == 1
    assert exit_stage_index(8, 8, 4) == 4
    assert exit_stage_index(3, 8, 4) == 2


def test_partition_stage_assignment():  # test_model.py:168-173
    cfg = ModelConfig(8, 16, 2, 32, 12, exits=(ExitSpec(2), ExitSpec(4)))
    part = partition(build_model(cfg, 0), 4)
    assert part.exit_stages() == [2, 3]
    assert part.stage_of_head("final") == 4


def test_partition_single_stage():  # test_model.py:176-181
    part = partition(build_model(small_config(exits=(ExitSpec(1),)), 0), 1)
    assert len(part.stages) == 1
    assert part.stages[0].has_embedding
    assert not part.tied_replicas


def test_partition_disjoint_cover():  # test_model.py:184-198
    cfg = small_config(exits=(ExitSpec(0), ExitSpec(2)), tie_embeddings=True)
    model = build_model(cfg, 0)
    part = partition(model, 2)
    seen = {}
    for st in part.stages:
        for name in st.params:
            seen.setdefault(name, []).append(st.index)
    assert set(seen) == set(model.params)
    for name, stages in seen.items():
        if len(stages) > 1:
            assert name in part.tied_replicas
            assert part.tied_replicas[name] == sorted(stages)
    assert part.tied_replicas == {"tok_emb": [1, 2]}


def test_partition_rejects_uneven_split():  # test_model.py:201-204
    with pytest.raises(ConfigError):
        partition(build_model(small_config(), 0), 3)


def test_build_is_deterministic():  # test_model.py:207-212
    cfg = small_config(exits=(ExitSpec(1, "mlp+embed"),))
    a, b = build_model(cfg, 123), build_model(cfg, 123)
    for name in a.params:
        assert np.array_equal(a.params[name].data, b.params[name].data)


def test_checkpoint_roundtrip_bit_exact(tmp_path):  # test_model.py:215-231
    cfg = small_config(exits=(ExitSpec(1, "norm+embed", 0.25), ExitSpec(3, "minimalistic", 0.5)),
                       tie_embeddings=True)
    model = build_model(cfg, 77)
    path = tmp_path / "model.ckpt"
    save_model(path, model)
    loaded = load_model(path)
    assert loaded.config == cfg
    assert set(loaded.params) == set(model.params)
    for name in model.params:
        assert np.array_equal(loaded.params[name].data, model.params[name].data)
    assert [h.key for h in loaded.heads] == [h.key for h in model.heads]
    save_model(tmp_path / "again.ckpt", loaded)
    assert (tmp_path / "again.ckpt").read_bytes() == path.read_bytes()


# ---- tests/test_inference.py: KV-cache discipline --------------------------------

def test_kvcache_monotone_fill():  # test_inference.py:82-90
    cache = KVCache([1, 2], max_positions=4, num_heads=2, head_dim=3, device="cpu")
    k = np.ones((2, 3))
    cache.fill(1, 0, k, k)
    with pytest.raises(ConfigError):
        cache.fill(1, 0, k * 2, k * 2)
    assert not cache.complete(1)
    cache.fill(2, 0, k, k)
    assert cache.complete(1)


def test_kvcache_rejects_unfilled_read():  # test_inference.py:93-98
    cache = KVCache([1], max_positions=4, num_heads=2, head_dim=3, device="cpu")
    cache.fill(1, 0, np.ones((2, 3)), np.ones((2, 3)))
    cache.view(1, 1)
    with pytest.raises(ConfigError):
        cache.view(1, 2)
