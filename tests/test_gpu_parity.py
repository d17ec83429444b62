"""GPU parity: the CUDA path (through the C-ABI) against the reference golden
vectors and the float64 oracle.

Tolerances (north star): fp32 parity mode — identical greedy tokens and exit
layers, confidences within 1e-5 relative; bf16 perf mode — exit-head
logits/confidence within 1e-3 relative (norm-wise for logits).
"""
import numpy as np
import pytest

import ee_oracle as O
from helpers import (arrays, c1_config, gold, mlp_config, oracle_inputs, small_config,
                     tap0_config)
from paper_2312_04916_b200 import inference as I
from paper_2312_04916_b200.errors import ConfigError, TokenError
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

pytestmark = pytest.mark.gpu

CONF_RTOL = 1e-5


@pytest.fixture(scope="module")
def c1():
    return build_model(c1_config(), 0)


@pytest.fixture(scope="module")
def small():
    return build_model(small_config(), 7)


def _close_conf(ours, ref, rtol=CONF_RTOL):
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):
        assert set(a) == set(b)
        for k in a:
            assert a[k] == pytest.approx(b[k], rel=rtol), (k, a[k], b[k])


def _same_decisions(tr, ref):
    assert tr.tokens == ref["tokens"]
    assert tr.exit_layers == ref["exit_layers"]


# ---- kernel-level parity on C1 (fp32) ----------------------------------------

def test_c1_prefill_taps_match_reference(c1):
    a = arrays()
    taps = I.prefill_taps(c1, gold()["c1_prompt"], dtype="fp32")
    for l in range(5):
        ref = a[f"c1_tap{l}"]
        err = np.abs(taps[l] - ref).max() / np.abs(ref).max()
        assert err < 1e-5, (l, err)


def test_c1_head_logits_match_reference(c1):
    a = arrays()
    for key, tap in (("exit_l1", 1), ("exit_l2", 2), ("final", 4)):
        ref = a[f"c1_logits_{key}"]
        lg, tok, conf, _ = I.head_logits(c1, key, a[f"c1_tap{tap}"][-1:], dtype="fp32")
        assert np.abs(lg[0] - ref).max() / np.abs(ref).max() < 1e-5
        _, rtok, rconf = O.exit_decision(ref, 1.0)
        assert tok[0] == rtok
        assert conf[0] == pytest.approx(rconf, rel=CONF_RTOL)


# ---- end-to-end generation parity -------------------------------------------

@pytest.mark.parametrize("tag,thr", [("thr08", 0.8), ("thr_force", 0.99 / 1024)])
def test_c1_kv_recompute_matches_reference(c1, tag, thr):
    ref = gold()[f"c1_{tag}"]
    tr = I.generate_kv_recompute(c1, gold()["c1_prompt"], thr, 8, dtype="fp32")
    _same_decisions(tr, ref)
    _close_conf(tr.confidences, ref["confidences"])
    assert tr.latencies == ref["latencies"]


def test_small_modes_match_reference_and_each_other(small):
    g = gold()
    prompt = g["small_prompts"][0]
    part = partition(small, 4)
    for run in g["small_runs"]:
        thr = run["threshold"]
        if "recompute" in run:
            tr = I.generate_kv_recompute(small, prompt, thr, 12, run["max_deferred"], dtype="fp32")
            _same_decisions(tr, run["recompute"])
            _close_conf(tr.confidences, run["recompute"]["confidences"])
            assert tr.latencies == run["recompute"]["latencies"]
        else:
            tr = I.generate_pipeline(part, prompt, thr, 12, dtype="fp32")
            _same_decisions(tr, run["pipeline"])
            assert tr.exit_stages == run["pipeline"]["exit_stages"]
            _close_conf(tr.confidences, run["pipeline"]["confidences"])
            assert tr.latencies == run["pipeline"]["latencies"]


def test_mixed_exit_layers_match_reference(small):
    g = gold()
    prompt = g["small_prompts"][0]
    part = partition(small, 4)
    for run in g["small_mixed"]:
        if "recompute" in run:
            tr = I.generate_kv_recompute(small, prompt, 0.015775, 16, run["max_deferred"],
                                         dtype="fp32")
            ref = run["recompute"]
        else:
            tr = I.generate_pipeline(part, prompt, 0.015775, 16, dtype="fp32")
            ref = run["pipeline"]
        _same_decisions(tr, ref)
        _close_conf(tr.confidences, ref["confidences"])


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_gpu_modes_bitwise_equal(small, dtype):
    """Row-stable kernels: pipeline and recompute agree BITWISE on the GPU
    (tokens, exit layers, confidence dicts), like the reference's own test
    (tests/test_inference.py:106-114)."""
    prompt = gold()["small_prompts"][0]
    part = partition(small, 4)
    for thr in (1.0, 6.0 / 64, 0.99 / 64, 0.015775):
        for md in (1, 2, 4):
            pipe = I.generate_pipeline(part, prompt, thr, 12, dtype=dtype)
            reco = I.generate_kv_recompute(small, prompt, thr, 12, md, dtype=dtype)
            assert pipe.tokens == reco.tokens
            assert pipe.exit_layers == reco.exit_layers
            assert pipe.confidences == reco.confidences


def test_greedy_reference_matches(small):
    g = gold()
    for p, ref in zip(g["small_prompts"], g["small_greedy"]):
        assert I.greedy_reference(small, p, 10, dtype="fp32") == ref
        assert I.generate_kv_recompute(small, p, 1.0, 10, dtype="fp32").tokens == ref


def test_mlp_and_tap0_heads(small):
    g = gold()
    mm = build_model(mlp_config(), 0)
    assert I.generate_kv_recompute(mm, [3, 1, 4], 1.0, 6, dtype="fp32").tokens == g["mlp_tokens"]
    tr = I.generate_kv_recompute(mm, [3, 1, 4], 0.99 / 64, 6, dtype="fp32")
    _same_decisions(tr, g["mlp_force"])
    _close_conf(tr.confidences, g["mlp_force"]["confidences"])
    tp = I.generate_pipeline(partition(mm, 2), [3, 1, 4], 0.99 / 64, 6, dtype="fp32")
    _same_decisions(tp, g["mlp_pipe_force"])
    mt = build_model(tap0_config(), 7)
    tr = I.generate_kv_recompute(mt, g["small_prompts"][0], 0.99 / 64, 10, dtype="fp32")
    _same_decisions(tr, g["tap0_reco"])
    _close_conf(tr.confidences, g["tap0_reco"]["confidences"])
    tp = I.generate_pipeline(partition(mt, 4), g["small_prompts"][0], 0.99 / 64, 10, dtype="fp32")
    _same_decisions(tp, g["tap0_pipe"])
    _close_conf(tp.confidences, g["tap0_pipe"]["confidences"])


def test_max_deferred_one_forces_full_fill(small):
    g = gold()["small_md1_14"]
    tr = I.generate_kv_recompute(small, gold()["small_prompts"][0], 0.99 / 64, 14, 1, dtype="fp32")
    _same_decisions(tr, g)
    full = max(tr.latencies)
    for i in range(1, len(tr.latencies) - 1):
        if tr.latencies[i] < full:
            assert tr.latencies[i + 1] == full


def test_errors(small):
    part = partition(small, 4)
    with pytest.raises(TokenError):
        I.generate_kv_recompute(small, [0] * 48, 1.0, 4)
    with pytest.raises(TokenError):
        I.generate_pipeline(part, [0] * 48, 1.0, 4)
    with pytest.raises(ConfigError):
        I.generate_kv_recompute(small, [], 1.0, 4)
    with pytest.raises(ConfigError):
        I.generate_kv_recompute(small, [1], 1.0, 4, max_deferred=0)
    with pytest.raises(ConfigError):
        I.generate_pipeline(partition(small, 1), [1, 2, 3], 1.0, 4)
    with pytest.raises(TokenError):
        I.generate_kv_recompute(small, [64], 1.0, 2)
    cfg = ModelConfig(4, 32, 4, 64, 32, exits=(ExitSpec(2, "layer+embed", 0.5),))
    with pytest.raises(ConfigError):
        I.generate_kv_recompute(build_model(cfg, 0), [1, 2], 1.0, 4)


def test_exit_decision_kats_on_gpu():
    fire, tok, conf = I.exit_decision(np.zeros(4), 0.25)
    assert conf == pytest.approx(0.25) and not fire and tok == 0
    z = np.zeros(8)
    z[3] = 30.0
    fire, tok, conf = I.exit_decision(z, 0.8)
    assert fire and tok == 3 and conf > 0.999999


# ---- row stability of the raw kernels ------------------------------------------

@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_head_kernel_row_stable(small, dtype):
    rng = np.random.default_rng(0)
    rows = rng.normal(size=(7, 32)).astype(np.float32)
    full = I.head_logits(small, "final", rows, dtype=dtype)
    for i in range(7):
        one = I.head_logits(small, "final", rows[i:i + 1], dtype=dtype)
        assert np.array_equal(full[0][i], one[0][0])
        assert full[1][i] == one[1][0] and full[2][i] == one[2][0]


# ---- bf16 at 7B width -------------------------------------------------------------

def test_bf16_exit_head_7b_width():
    """Exit-head logits/confidence at h=4096, V=50304 in bf16 within 1e-3
    relative of the float64 oracle (weights and rows rounded to bf16 first,
    so the tolerance measures the kernel, not the input rounding)."""
    import torch
    cfg = ModelConfig(1, 4096, 32, 50304, 16, exits=(ExitSpec(1, "minimalistic", 0.1),))
    m = build_model(cfg, 0, init="device", dtype=torch.bfloat16)
    rng = np.random.default_rng(3)
    rows = (rng.normal(size=(5, 4096)) * 1.0).astype(np.float32)
    lg, tok, conf, _ = I.head_logits(m, "exit_l1", rows, dtype="bf16")
    W = m.params["exit_l1.out"].data.float().cpu().numpy().astype(np.float64)
    xb = torch.from_numpy(rows).bfloat16().float().numpy().astype(np.float64)
    ref = xb @ W.T
    rel = np.linalg.norm(lg - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-3, rel
    for i in range(5):
        _, rtok, rconf = O.exit_decision(ref[i], 1.0)
        assert conf[i] == pytest.approx(rconf, rel=1e-3)
        if tok[i] != rtok:  # near-tie: report, allowed only within tolerance
            assert abs(ref[i][tok[i]] - ref[i][rtok]) < 1e-3 * abs(ref[i][rtok])


def test_fp32_generation_at_7b_width_matches_reference():
    """SURVEY Appendix B.3 at real width: a 2-layer h=4096 / V=50304 model with
    the reference's float64 initialisation (`build_model(cfg, 0)`, identical
    draws) decoded by the GPU path in fp32 parity mode: identical tokens and
    exit layers to the reference (tests/golden/golden_7b.json, made by
    tests/golden/make_7b_slice.py), at threshold 1.0 and at 0.05 (early exits
    and deferred recomputation at real width); confidences within 1e-4
    relative (fp32 dot products of length 4096 / softmax over 50304 against
    float64)."""
    import json
    import os
    from helpers import GOLD_DIR
    with open(os.path.join(GOLD_DIR, "golden_7b.json")) as f:
        g = json.load(f)
    cfg = ModelConfig(2, 4096, 32, 50304, 2048, exits=(ExitSpec(1, "minimalistic", 0.1),))
    m = build_model(cfg, 0)
    for key, thr in (("thr1", 1.0), ("thr005", 0.05)):
        tr = I.generate_kv_recompute(m, g["prompt"], thr, 6, dtype="fp32")
        _same_decisions(tr, g[key])
        _close_conf(tr.confidences, g[key]["confidences"], rtol=1e-4)


@pytest.mark.parametrize("n", [17, 40, 100])
def test_bf16_prefill_gemm_matches_gemv_and_oracle(n):
    """Passes with more than 16 rows (prompt prefill) run the tcgen05 GEMM
    over the tiled weights (csrc/prefill_gemm.cu) instead of the GEMV.
    Causal attention makes the first 16 rows of an n-row prefill independent
    of the later rows, so they are compared with a 16-row prefill (GEMV
    path): hidden states at every tap within 1e-2 relative (bf16 weights and
    activations, different fp32 accumulation order); the full n rows are also
    checked against the float64 oracle run on the bf16-rounded weights
    (2e-2 relative per tap)."""
    import torch
    cfg = ModelConfig(3, 512, 4, 96, 128, exits=(ExitSpec(1, "minimalistic", 0.3),))
    host = build_model(cfg, 5)
    dev = {k: torch.from_numpy(p.data).to("cuda").bfloat16() for k, p in host.params.items()}
    from paper_2312_04916_b200.model import model_from_arrays
    m = model_from_arrays(cfg, dev)
    toks = [int(t) for t in np.random.default_rng(n).integers(0, 96, size=n)]
    big = I.prefill_taps(m, toks, dtype="bf16")
    small = I.prefill_taps(m, toks[:16], dtype="bf16")
    for l in range(4):
        a, b = big[l][:16], small[l]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-2, l
    P = {k: v.float().cpu().numpy().astype(np.float64) for k, v in dev.items()}
    kv = O.KV(range(1, 4), cfg.max_seq_len, cfg.num_heads, cfg.hidden_dim // cfg.num_heads)
    x = O.embed(P, cfg.vocab_size, toks, range(n))
    for l in range(1, 4):
        x = O.layer_step(P, l, x, list(range(n)), kv, cfg.num_heads)
        err = np.linalg.norm(big[l] - x) / np.linalg.norm(x)
        assert err < 2e-2, (l, err)


def test_tiled_bf16_modes_bitwise_equal():
    """Row-stability of the perf path itself (tiled bf16 weights: TMA-fed
    stream-K GEMV, folded RMSNorm, split-KV attention, tiled exit head): the
    pipeline (one row per message) and KV-recompute (deferred rows batched,
    up to 5 per pass) modes agree bitwise on tokens, exit layers and
    confidences at h = 512 across thresholds that force early exits."""
    import torch
    cfg = ModelConfig(4, 512, 4, 256, 64, exits=(ExitSpec(1, "minimalistic", 0.3),
                                                 ExitSpec(2, "minimalistic", 0.6)))
    m = build_model(cfg, 11, init="device", dtype=torch.bfloat16)
    part = partition(m, 2, copy=False)
    prompt = [int(t) for t in np.random.default_rng(4).integers(0, 256, size=7)]
    for thr in (1.0, 0.99 / 256, 1.2 / 256, 2.0 / 256):
        for md in (1, 4):
            reco = I.generate_kv_recompute(m, prompt, thr, 20, md)
            pipe = I.generate_pipeline(part, prompt, thr, 20)
            assert reco.tokens == pipe.tokens, thr
            assert reco.exit_layers == pipe.exit_layers, thr
            assert reco.confidences == pipe.confidences, thr


def test_tiled_modes_bitwise_equal_with_many_deferred_rows():
    """max_deferred = 20 makes recompute passes of up to 21 rows (more than the
    16-row GEMV tile): decode passes must still take the row-stable GEMV
    (only the prompt prefill may use the multi-row tcgen05 GEMM), so pipeline
    (one row per message) and recompute agree bitwise; norm+embed and
    mlp+embed heads on the tiled bf16 path."""
    import torch
    cfg = ModelConfig(4, 512, 4, 256, 64, exits=(ExitSpec(1, "norm+embed", 0.3),
                                                 ExitSpec(2, "mlp+embed", 0.6)))
    m = build_model(cfg, 13, init="device", dtype=torch.bfloat16)
    part = partition(m, 2, copy=False)
    prompt = [int(t) for t in np.random.default_rng(8).integers(0, 256, size=20)]
    for thr in (0.99 / 256, 1.5 / 256):
        reco = I.generate_kv_recompute(m, prompt, thr, 30, 20)
        pipe = I.generate_pipeline(part, prompt, thr, 30)
        assert reco.tokens == pipe.tokens, thr
        assert reco.exit_layers == pipe.exit_layers, thr
        assert reco.confidences == pipe.confidences, thr
        assert any(e < 4 for e in reco.exit_layers)


@pytest.mark.parametrize("prompt_len,max_new,max_deferred", [(250, 40, 15), (1900, 140, 3)])
def test_tiled_modes_bitwise_equal_long_context(prompt_len, max_new, max_deferred):
    """Pipeline (one row per pass) and KV recomputation (up to 16 rows per
    pass) agree bitwise when rows cross the 256-position attention chunk
    boundary (ordered cross-chunk merge) and near the 2048-position limit
    (8 chunks)."""
    import torch
    cfg = ModelConfig(2, 512, 4, 256, 2048, exits=(ExitSpec(1, "minimalistic", 0.3),))
    m = build_model(cfg, 17, init="device", dtype=torch.bfloat16)
    part = partition(m, 2, copy=False)
    prompt = [int(t) for t in np.random.default_rng(prompt_len).integers(0, 256, size=prompt_len)]
    for thr in (1.0, 1.3 / 256):
        reco = I.generate_kv_recompute(m, prompt, thr, max_new, max_deferred)
        pipe = I.generate_pipeline(part, prompt, thr, max_new)
        assert reco.tokens == pipe.tokens, thr
        assert reco.exit_layers == pipe.exit_layers, thr
        assert reco.confidences == pipe.confidences, thr


def test_bridge_runs_reference_model_objects(c1):
    """`eepipe_bridge`: a model object with the reference's surface (`config`
    with the reference fields, `named_arrays()` of float64 arrays) decodes on
    the GPU through the bridge with the reference's own golden tokens, exit
    layers and confidences (C1, threshold 0.8), and re-partitions for
    pipeline mode (tokens equal to the recompute run)."""
    from types import SimpleNamespace
    from paper_2312_04916_b200 import eepipe_bridge as B
    cfg = c1.config
    ref_like = SimpleNamespace(
        config=SimpleNamespace(num_layers=cfg.num_layers, hidden_dim=cfg.hidden_dim,
                               num_heads=cfg.num_heads, vocab_size=cfg.vocab_size,
                               max_seq_len=cfg.max_seq_len, tie_embeddings=cfg.tie_embeddings,
                               exits=tuple(SimpleNamespace(layer_index=e.layer_index,
                                                           head_kind=e.head_kind,
                                                           loss_weight=e.loss_weight)
                                           for e in cfg.exits)),
        named_arrays=c1.named_arrays)
    ref = gold()["c1_thr08"]
    tr = B.generate_kv_recompute(ref_like, gold()["c1_prompt"], 0.8, 8)
    _same_decisions(tr, ref)
    _close_conf(tr.confidences, ref["confidences"])
    # a reference-surface StagePartition: config + stages holding their params
    part = partition(c1, 2)
    part_like = SimpleNamespace(config=ref_like.config, num_stages=2,
                                stages=[SimpleNamespace(params=st.params) for st in part.stages])
    pipe = B.generate_pipeline(part_like, gold()["c1_prompt"], 0.8, 8)
    assert pipe.tokens == tr.tokens and pipe.exit_layers == tr.exit_layers
