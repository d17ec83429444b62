"""Shared test helpers: golden fixtures and model <-> oracle plumbing."""
import json
import os

import numpy as np

GOLD_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_gold = None
_arrays = None


def gold():
    global _gold
    if _gold is None:
        with open(os.path.join(GOLD_DIR, "golden.json")) as f:
            _gold = json.load(f)
    return _gold


def arrays():
    global _arrays
    if _arrays is None:
        _arrays = dict(np.load(os.path.join(GOLD_DIR, "golden.npz")))
    return _arrays


def oracle_inputs(model):
    """(params dict of f64 arrays, oracle Cfg, oracle heads) for a host model."""
    import ee_oracle as O
    c = model.config
    P = {n: p.data for n, p in model.params.items()}
    return P, O.Cfg(c.num_layers, c.hidden_dim, c.num_heads, c.vocab_size, c.max_seq_len), \
        O.heads_of(model.heads)


def c1_config():
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    return ModelConfig(4, 256, 4, 1024, 128, exits=(ExitSpec(1, "minimalistic", 0.25),
                                                    ExitSpec(2, "minimalistic", 0.5)))


def small_config():
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    return ModelConfig(8, 32, 4, 64, 48, exits=(ExitSpec(2, loss_weight=0.3),
                                                ExitSpec(4, loss_weight=0.6)))


def mlp_config():
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    return ModelConfig(4, 32, 4, 64, 32, exits=(ExitSpec(2, "mlp+embed", 0.5),))


def tap0_config():
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    return ModelConfig(8, 32, 4, 64, 48, exits=(ExitSpec(0, loss_weight=0.2),
                                                ExitSpec(4, loss_weight=0.5)))


def params_digest(model):
    import hashlib
    h = hashlib.sha256()
    for name in sorted(model.params):
        h.update(name.encode())
        h.update(np.ascontiguousarray(model.params[name].data).tobytes())
    return h.hexdigest()
