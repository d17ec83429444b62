"""Reference-side bridge (`paper_2312_04916_b200/eepipe_bridge.py`): a
reference `EarlyExitModel` converts parameter for parameter.  Against the
real reference package when it is importable (this container:
/root/reference/pkg/src), else against a stand-in with the reference's
attribute surface (`config` with the reference fields, `named_arrays()`)."""
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2312_04916_b200 import eepipe_bridge as B
from paper_2312_04916_b200.errors import ConfigError
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model

REF_SRC = "/root/reference/pkg/src"


def _reference_model(cfg_args, seed):
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, REF_SRC)
    try:
        import eepipe.model as R
    finally:
        sys.path.remove(REF_SRC)
    n, h, nh, V, s, exits, tied = cfg_args
    return R.build_model(R.ModelConfig(n, h, nh, V, s, exits=tuple(R.ExitSpec(*e) for e in exits),
                                       tie_embeddings=tied), seed)


@pytest.mark.parametrize("cfg_args,seed", [
    ((4, 256, 4, 1024, 128, ((1, "minimalistic", 0.25), (2, "minimalistic", 0.5)), False), 0),
    ((6, 32, 4, 64, 32, ((0, "norm+embed", 0.1), (2, "mlp+embed", 0.3), (3, "layer+embed", 0.5)),
      True), 3),
])
def test_reference_model_converts_bitwise(cfg_args, seed):
    ref = _reference_model(cfg_args, seed)
    ours = B.model_from_reference(ref)
    mine = build_model(B.config_from_reference(ref.config), seed)
    assert ours.config == mine.config
    assert [(h.key, h.kind, h.layer_index) for h in ours.heads] == \
        [(h.key, h.kind, h.layer_index) for h in mine.heads]
    ra = ref.named_arrays()
    assert set(ra) == set(ours.params)
    for name, arr in ra.items():
        assert isinstance(ours.params[name].data, np.ndarray), name
        assert np.array_equal(ours.params[name].data, arr), name
        assert np.array_equal(mine.params[name].data, arr), name


def test_stand_in_model_converts_and_validates():
    cfg = ModelConfig(2, 32, 4, 64, 16, exits=(ExitSpec(1, "minimalistic", 0.5),))
    m = build_model(cfg, 1)
    ref_like = SimpleNamespace(
        config=SimpleNamespace(num_layers=2, hidden_dim=32, num_heads=4, vocab_size=64,
                               max_seq_len=16, tie_embeddings=False,
                               exits=(SimpleNamespace(layer_index=1, head_kind="minimalistic",
                                                      loss_weight=0.5),)),
        named_arrays=m.named_arrays)
    conv = B.model_from_reference(ref_like)
    assert conv.config == cfg
    arrs = m.named_arrays()
    arrs.pop("final.norm")
    ref_like.named_arrays = lambda: arrs
    with pytest.raises(ConfigError, match="missing parameter final.norm"):
        B.model_from_reference(ref_like)


def test_reference_partition_rebuilds_model():
    ref = _reference_model((6, 32, 4, 64, 32, ((2, "minimalistic", 0.3),), True), 4)
    sys.path.insert(0, REF_SRC)
    try:
        import eepipe.model as R
    finally:
        sys.path.remove(REF_SRC)
    part = R.partition(ref, 3)
    ours = B.model_from_reference_partition(part)
    for name, arr in ref.named_arrays().items():
        assert np.array_equal(ours.params[name].data, arr), name
