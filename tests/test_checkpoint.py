"""Checkpoint bridge: the reference's EEPIPE-CKPT v1
format (`eepipe/checkpoint.py`) read and written by
`paper_2312_04916_b200.checkpoint`, pinned against a checkpoint the reference
itself wrote (`tests/golden/trained_tiny.ckpt`, made by
`tests/golden/make_trained.py`), and the oracle pinned against the reference's
traces of that trained model (non-trivial early exits at 0.8 / 0.9).  CPU only.
"""
import json
import os
import struct

import numpy as np
import pytest

import ee_oracle as O
from helpers import GOLD_DIR, oracle_inputs, params_digest
from paper_2312_04916_b200 import checkpoint as C
from paper_2312_04916_b200.errors import ConfigError
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model

CKPT = os.path.join(GOLD_DIR, "trained_tiny.ckpt")


def trained_gold():
    with open(os.path.join(GOLD_DIR, "trained.json")) as f:
        return json.load(f)


def test_load_reference_checkpoint_bitwise():
    m = C.load_model(CKPT)
    g = trained_gold()
    assert params_digest(m) == g["digest"]
    assert m.config == ModelConfig(4, 64, 4, 128, 64, exits=(ExitSpec(1, "minimalistic", 0.25),
                                                              ExitSpec(2, "minimalistic", 0.5)))
    assert [h.key for h in m.heads] == ["exit_l1", "exit_l2", "final"]


def test_save_reproduces_reference_bytes(tmp_path):
    m = C.load_model(CKPT)
    out = tmp_path / "rt.ckpt"
    C.save_model(out, m)
    assert out.read_bytes() == open(CKPT, "rb").read()


def test_round_trip_random_init_and_tied(tmp_path):
    g = trained_gold()
    cfg = ModelConfig(4, 64, 4, 128, 64, exits=(ExitSpec(1, "minimalistic", 0.25),
                                                 ExitSpec(2, "minimalistic", 0.5)))
    m = build_model(cfg, 0)
    assert params_digest(m) == g["init_digest"]
    C.save_model(tmp_path / "a.ckpt", m)
    m2 = C.load_model(tmp_path / "a.ckpt")
    assert params_digest(m2) == params_digest(m)
    tied = ModelConfig(4, 32, 4, 64, 16, exits=(ExitSpec(1, loss_weight=0.25),
                                                 ExitSpec(2, "mlp+embed", 0.5)),
                       tie_embeddings=True)
    mt = build_model(tied, 3)
    C.save_model(tmp_path / "t.ckpt", mt)
    mt2 = C.load_model(tmp_path / "t.ckpt")
    assert mt2.config == tied
    assert params_digest(mt2) == params_digest(mt)
    assert mt2.heads[0].param_names["out"] == "tok_emb"


def test_corrupt_checkpoints_raise_config_error(tmp_path):
    raw = open(CKPT, "rb").read()
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOT-A-CKPT\0\0" + raw[12:])
    with pytest.raises(ConfigError, match="magic"):
        C.load_model(bad)
    bad.write_bytes(raw[:12] + struct.pack("<I", 2) + raw[16:])
    with pytest.raises(ConfigError, match="version"):
        C.load_model(bad)
    bad.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(ConfigError):
        C.load_model(bad)


def test_oracle_reproduces_reference_on_trained_model():
    """The oracle (test infrastructure) restates the reference bitwise on the
    trained checkpoint as well, including the early-exit-heavy runs."""
    m = C.load_model(CKPT)
    P, cfg, heads = oracle_inputs(m)
    g = trained_gold()
    early = 0
    for run in g["runs"]:
        prompt = g["prompts"][run["prompt"]]
        if "recompute" in run:
            tr = O.generate_kv_recompute(P, cfg, heads, prompt, run["threshold"], 24,
                                         run["max_deferred"])
            ref = run["recompute"]
        else:
            tr = O.generate_pipeline(P, cfg, heads, 2, prompt, run["threshold"], 24)
            ref = run["pipeline"]
            assert tr["exit_stages"] == ref["exit_stages"]
        assert tr["tokens"] == ref["tokens"]
        assert tr["exit_layers"] == ref["exit_layers"]
        assert tr["confidences"] == ref["confidences"]
        early += sum(1 for e in ref["exit_layers"] if e < cfg.L)
    assert early > 100  # the fixture really exercises early exits
