"""bf16 PERF-PATH parity: the kernels `bench.py` times (tiled bf16 weights,
TMA-fed GEMV chain with folded RMSNorm and the QKV/KV-write epilogue,
split-KV decode attention, tiled exit head) against the float64 oracle and
the REFERENCE run on the same bf16-rounded weights.

1. One decode layer at a time at 7B width (h = 4096, 32 heads of 128) for
   m = 1, 2, 5 rows with permuted positions after a 40-row prompt, against
   `ee_oracle.layer_step` (eepipe/inference.py:216-229) fed the GPU's own
   input rows and KV prefix, on the bf16-rounded weights.  Tolerances are the
   bf16 ones: the perf path rounds the normalised input, the attention output
   and the GELU output to bf16 (unit roundoff u = 2^-9) before each GEMV and
   stores K/V in bf16, so each layer's update (x_out - x_in) carries a
   norm-wise relative error of a few u (measured 2-4e-3); the tests allow
   1.5e-2 on the update and 8e-3 on the new K/V rows (one bf16 rounding on
   top of the q/k/v error).
2. End-to-end bf16 generation against the reference's own traces on the
   bf16-rounded weights (tests/golden/make_bf16_golden.py): the 7B-width
   2-layer slice of SURVEY B.3 (2 prompts x thresholds 1.0/0.3/0.1/0.05,
   KV recompute + pipeline) and the reference-trained checkpoint (3 prompts x
   0.9/0.8/0.5, both modes).  Tokens and exit layers must be identical until
   a decision whose confidence lies within CONF_TOL of the threshold (or a
   greedy token whose reference probability is within CONF_TOL of the
   reference's maximum -- an argmax near-tie, checked against the top-5 the
   fixture records at every reference decision) flips; a
   run is compared up to that point, every such mismatch is printed, and any
   other divergence fails.  Confidences of compared tokens: 5e-2 relative
   (the end-to-end bf16 band derived at CONF_RTOL; the head kernel alone is
   within 1e-3 of the oracle, tests/test_gpu_parity.py).
"""
import json
import os

import numpy as np
import pytest

import ee_oracle as O
from helpers import GOLD_DIR
from paper_2312_04916_b200 import checkpoint as C
from paper_2312_04916_b200 import inference as I
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

pytestmark = pytest.mark.gpu

UPDATE_RTOL = 1.5e-2
KV_RTOL = 8e-3
# End to end, a token's hidden state has passed every layer with bf16
# activations and a bf16 KV cache (update error ~3.5e-3 per layer, test 1),
# so its logits carry an absolute error of ~1e-2 at 7B width and the max
# softmax probability a relative error of ~1e-2 (measured up to 3.1e-2
# after 12 tokens); 5e-2 bounds it.  A decision may flip only where the
# reference confidence lies within that same band around the threshold.
CONF_TOL = 5e-2       # relative: a decision this close to the threshold may flip
CONF_RTOL = 5e-2      # bf16 confidences vs the reference on bf16 weights


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def wide():
    import torch
    cfg = ModelConfig(2, 4096, 32, 512, 2048, exits=(ExitSpec(1, "minimalistic", 0.1),))
    m = build_model(cfg, 0, init="device", dtype=torch.bfloat16)
    P = {k: p.data.float().cpu().double().numpy() for k, p in m.params.items()
         if k.startswith("layer")}
    return m, P


@pytest.mark.parametrize("positions", [[40], [41, 40], [43, 40, 44, 41, 42]])
def test_tiled_decode_layer_chain_7b_width(wide, positions):
    import torch
    m, P = wide
    cfg = m.config
    h, nh = cfg.hidden_dim, cfg.num_heads
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, cfg.vocab_size, 40)]
    I.prefill_taps(m, prompt, dtype="bf16")  # fills layers 1-2 at positions 0..39
    eng = I._engine_for(m, m.params, m.heads, cfg, range(1, 3), True, "bf16")
    assert eng.tiled
    n = len(positions)
    toks = [int(t) for t in np.random.default_rng(n).integers(0, cfg.vocab_size, n)]
    rows = (m.params["tok_emb"].data[toks].float() +
            m.params["pos_emb"].data[positions].float()).cpu().numpy()
    kv = O.KV([1, 2], cfg.max_seq_len, nh, h // nh)
    with torch.cuda.device(eng.device), torch.cuda.stream(eng.stream):
        eng._grow(n)
        eng.x[:n].copy_(torch.from_numpy(rows))
        eng.refresh_stats(0, n)
        eng.upload_ctrl(list(positions))
        x_in = rows.astype(np.float64)
        for slot, layer in enumerate((1, 2)):
            kc = eng.kv.k(layer)[:40].float().cpu().double().numpy()
            vc = eng.kv.v(layer)[:40].float().cpu().double().numpy()
            for p in range(40):
                kv.fill(layer, p, kc[p].reshape(nh, -1), vc[p].reshape(nh, -1))
            eng.run_layers(slot, slot + 1, n, [n], max(positions), 0)
            x_gpu = eng.x[:n].cpu().double().numpy()
            x_ref = O.layer_step(P, layer, x_in, positions, kv, nh)
            err = _rel(x_gpu - x_in, x_ref - x_in)
            print(f"layer {layer} m={n}: update rel err {err:.2e}")
            assert err < UPDATE_RTOL, (layer, err)
            for r, p in enumerate(positions):
                kg = eng.kv.k(layer)[p].float().cpu().double().numpy()
                vg = eng.kv.v(layer)[p].float().cpu().double().numpy()
                assert _rel(kg, kv.k[layer][p].reshape(-1)) < KV_RTOL, (layer, p)
                assert _rel(vg, kv.v[layer][p].reshape(-1)) < KV_RTOL, (layer, p)
            x_in = x_gpu  # the next layer is checked on the GPU's own input


def _near(ref_conf, thr, tol):
    return any(abs(c - thr) <= tol * thr for c in ref_conf.values())


def compare_trace(tr, ref, thr, *, stages=False, label="", conf_tol=CONF_TOL,
                  conf_rtol=CONF_RTOL):
    """Tokens / exit layers identical up to the first near-threshold (or
    near-tie) flip.  Returns (compared tokens, mismatch report or None)."""
    n = len(ref["tokens"])
    for i in range(n):
        same = (tr.tokens[i] == ref["tokens"][i] and tr.exit_layers[i] == ref["exit_layers"][i]
                and (not stages or tr.exit_stages[i] == ref["exit_stages"][i]))
        rc = ref["confidences"][i]
        if not same:
            near_thr = _near(rc, thr, conf_tol)
            # argmax near-tie: same exit layer, and our token is within
            # CONF_TOL of the maximum of the REFERENCE's own distribution at
            # the deciding head (its top-5 is recorded with every reference
            # exit_decision call, tests/golden/make_bf16_golden.py)
            tie = tr.exit_layers[i] == ref["exit_layers"][i] and any(
                d["token"] == ref["tokens"][i] and any(
                    t == tr.tokens[i] and pr >= (1.0 - conf_tol) * d["top5"][0][1]
                    for t, pr in d["top5"]) for d in ref.get("decisions", ()))
            rep = {"run": label, "token": i, "threshold": thr,
                   "ours": [tr.tokens[i], tr.exit_layers[i]],
                   "reference": [ref["tokens"][i], ref["exit_layers"][i]],
                   "reference_conf": rc, "our_conf": tr.confidences[i],
                   "kind": "near-threshold" if near_thr else ("argmax near-tie" if tie else "BAD")}
            assert near_thr or tie, rep
            return i, rep
        for k, c in rc.items():
            dev = abs(tr.confidences[i][k] - c) / c
            compare_trace.max_dev = max(getattr(compare_trace, "max_dev", 0.0), dev)
            assert dev <= conf_rtol, (label, i, k, tr.confidences[i][k], c)
    return n, None


def _run_fixture(model, g, part_stages=2):
    part = partition(model, part_stages, copy=False)
    compared, total, reports = 0, 0, []
    for run in g["runs"]:
        prompt = g["prompts"][run["prompt"]]
        thr = run["threshold"]
        new = len(run["tokens"])
        if run["mode"] == "recompute":
            tr = I.generate_kv_recompute(model, prompt, thr, new, run["max_deferred"],
                                         dtype="bf16")
        else:
            tr = I.generate_pipeline(part, prompt, thr, new, dtype="bf16")
        label = f"{run['mode']} prompt {run['prompt']} thr {thr}"
        n, rep = compare_trace(tr, run, thr, stages=run["mode"] == "pipeline", label=label)
        compared += n
        total += new
        if rep:
            reports.append(rep)
    for r in reports:
        print("bf16 exit-decision mismatch (reported):", r)
    print(f"compared {compared}/{total} tokens; max relative confidence deviation "
          f"{getattr(compare_trace, 'max_dev', 0.0):.2e}")
    return compared, total, reports


def test_bf16_generation_7b_width_matches_reference_on_bf16_weights():
    import torch
    with open(os.path.join(GOLD_DIR, "golden_7b_bf16.json")) as f:
        g = json.load(f)
    L, h, nh, V, s_max, tap = g["config"]
    cfg = ModelConfig(L, h, nh, V, s_max, exits=(ExitSpec(tap, "minimalistic", 0.1),))
    host = build_model(cfg, 0)
    dev = {k: torch.from_numpy(p.data).to("cuda").bfloat16() for k, p in host.params.items()}
    del host
    from paper_2312_04916_b200.model import model_from_arrays
    m = model_from_arrays(cfg, dev)
    compared, total, reports = _run_fixture(m, g)
    early = sum(1 for run in g["runs"] for e in run["exit_layers"] if e < L)
    assert early >= 10  # the fixture exercises early exits at real width
    assert compared >= 0.75 * total, (compared, total)


def test_bf16_trained_checkpoint_matches_reference_on_bf16_weights():
    import torch
    with open(os.path.join(GOLD_DIR, "trained_bf16.json")) as f:
        g = json.load(f)
    host = C.load_model(os.path.join(GOLD_DIR, "trained_tiny.ckpt"))
    dev = {k: torch.from_numpy(p.data).to("cuda").bfloat16() for k, p in host.params.items()}
    from paper_2312_04916_b200.model import model_from_arrays
    m = model_from_arrays(host.config, dev)
    compared, total, reports = _run_fixture(m, g)
    assert compared >= 0.75 * total, (compared, total)
