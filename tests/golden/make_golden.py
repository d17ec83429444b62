"""Generate golden vectors from the REFERENCE implementation (run in the build
container only; `/root/reference` does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python \
        python tests/golden/make_golden.py

Imports `eepipe` from `/root/reference/pkg/src` with the numpy backend
(``EEPIPE_BACKEND=python``; the backend choice is recorded in the fixture) and
writes `tests/golden/golden.json` + `tests/golden/golden.npz`.  The oracle
(`oracle/ee_oracle.py`) is pinned against these in
`tests/test_oracle_golden.py`; the GPU path is checked against them and the
oracle in `tests/test_gpu_parity.py`.

Fixtures:
  * c1_*: the C1 tiny model (L=4, h=256, nh=4, V=1024, s_max=128, exits at 1
    and 2), seed 0, prompt default_rng(1).integers(0,1024,8): KV-recompute
    traces at thr 0.8 and 0.99/1024 (8 new tokens), per-tap hidden states of
    the prefill and every head's logits at the last prompt row.
  * small_*: the reference test model ModelConfig(8,32,4,64,48, exits 2:0.3,
    4:0.6), seed 7, prompt default_rng(17) length 6 (tests/test_inference.py
    :25-39): both modes over thr {1.0, 6/64, 0.99/64} x max_deferred {1,2,4},
    12 tokens, P=4; greedy_reference for 2 prompts x 10 tokens.
  * mlp_*: mlp+embed head model (tests/test_inference.py:226-233).
  * tap0_*: exit at tap 0 (quirk 1 of SURVEY §8c).
  * ce_*: exit-head training KATs: logits/CE/grads via the reference autodiff
    (`run_head` + `cross_entropy` + `Tape.backward`), minimalistic and
    norm+embed, n=24, h=32, V=96.
  * wl_*: `single_device_gradients` for a tiny tied model (per-exit losses and
    a few gradient checksums) — training parity anchor.
"""

import hashlib
import json
import os
import sys

import numpy as np

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import eepipe  # noqa: E402
from eepipe import kernels  # noqa: E402
from eepipe.autodiff import Tape, Tensor, cross_entropy  # noqa: E402
from eepipe.inference import (  # noqa: E402
    KVCache, _InferParams, _layer_step, generate_kv_recompute, generate_pipeline,
    greedy_reference)
from eepipe.model import (  # noqa: E402
    ExitSpec, ModelConfig, build_model, partition, run_head)
from eepipe.pipeline import single_device_gradients  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def trace_dict(tr):
    return {"tokens": [int(t) for t in tr.tokens], "exit_layers": list(tr.exit_layers),
            "exit_stages": list(tr.exit_stages),
            "confidences": [{k: float(v) for k, v in c.items()} for c in tr.confidences],
            "latencies": [float(x) for x in tr.latencies],
            "total_latency": float(tr.total_latency),
            "baseline_latency": float(tr.baseline_latency)}


def params_digest(model):
    h = hashlib.sha256()
    for name in sorted(model.params):
        h.update(name.encode())
        h.update(np.ascontiguousarray(model.params[name].data).tobytes())
    return h.hexdigest()


def main():
    gold = {"backend": kernels.BACKEND, "eepipe_version": eepipe.__version__}
    arrays = {}

    # ---- C1 tiny ---------------------------------------------------------
    c1 = ModelConfig(4, 256, 4, 1024, 128,
                     exits=(ExitSpec(1, "minimalistic", 0.25), ExitSpec(2, "minimalistic", 0.5)))
    m1 = build_model(c1, 0)
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, 1024, size=8)]
    gold["c1_prompt"] = prompt
    gold["c1_digest"] = params_digest(m1)
    gold["c1_tok_emb_0_4"] = [float(v) for v in m1.params["tok_emb"].data[0, :4]]
    for tag, thr in (("thr08", 0.8), ("thr_force", 0.99 / 1024)):
        gold[f"c1_{tag}"] = trace_dict(generate_kv_recompute(m1, prompt, thr, 8))
    # per-tap prefill hidden states + head logits at the last prompt row
    ip = _InferParams(m1.params, m1.heads, c1, range(1, 5), True)
    cache = KVCache(range(1, 5), c1.max_seq_len, c1.num_heads, c1.hidden_dim // c1.num_heads)
    x = ip.embed(prompt, range(8))
    arrays["c1_tap0"] = x
    for l in range(1, 5):
        x = _layer_step(ip.layers[l], x, list(range(8)), cache, l, c1.num_heads)
        arrays[f"c1_tap{l}"] = x
    for hd, mats in ip.heads:
        arrays[f"c1_logits_{hd.key}"] = ip.head_logits(hd, mats, arrays[f"c1_tap{hd.layer_index}"][-1])

    # ---- small reference test model ---------------------------------------
    cs = ModelConfig(8, 32, 4, 64, 48,
                     exits=(ExitSpec(2, loss_weight=0.3), ExitSpec(4, loss_weight=0.6)))
    ms = build_model(cs, 7)
    ps = partition(ms, 4)
    rng = np.random.default_rng(17)
    prompts = [[int(t) for t in rng.integers(0, 64, size=6)] for _ in range(3)]
    gold["small_prompts"] = prompts
    gold["small_digest"] = params_digest(ms)
    runs = []
    for thr in (1.0, 6.0 / 64, 0.99 / 64):
        for md in (1, 2, 4):
            reco = generate_kv_recompute(ms, prompts[0], thr, 12, md)
            runs.append({"threshold": thr, "max_deferred": md, "recompute": trace_dict(reco)})
        pipe = generate_pipeline(ps, prompts[0], thr, 12)
        runs.append({"threshold": thr, "pipeline": trace_dict(pipe)})
    gold["small_runs"] = runs
    # a threshold inside the confidence spread gives a mix of exit layers
    # (2, 4 and 8) within one sequence; 0.015775 sits in a gap of the
    # thr=1.0 confidence distribution (~6e-4 relative from its neighbours)
    mixed = []
    for md in (1, 2, 4):
        mixed.append({"max_deferred": md, "recompute": trace_dict(
            generate_kv_recompute(ms, prompts[0], 0.015775, 16, md))})
    mixed.append({"pipeline": trace_dict(generate_pipeline(ps, prompts[0], 0.015775, 16))})
    gold["small_mixed"] = mixed
    gold["small_greedy"] = [greedy_reference(ms, p, 10) for p in prompts[:2]]
    # max_deferred=1 run with 14 tokens (tests/test_inference.py:137-147)
    gold["small_md1_14"] = trace_dict(generate_kv_recompute(ms, prompts[0], 0.99 / 64, 14, 1))

    # ---- mlp+embed head ----------------------------------------------------
    cm = ModelConfig(4, 32, 4, 64, 32, exits=(ExitSpec(2, "mlp+embed", 0.5),))
    mm = build_model(cm, 0)
    gold["mlp_digest"] = params_digest(mm)
    gold["mlp_tokens"] = generate_kv_recompute(mm, [3, 1, 4], 1.0, 6).tokens
    gold["mlp_force"] = trace_dict(generate_kv_recompute(mm, [3, 1, 4], 0.99 / 64, 6))
    gold["mlp_pipe_force"] = trace_dict(generate_pipeline(partition(mm, 2), [3, 1, 4], 0.99 / 64, 6))

    # ---- tap-0 exit quirk ---------------------------------------------------
    ct = ModelConfig(8, 32, 4, 64, 48, exits=(ExitSpec(0, loss_weight=0.2), ExitSpec(4, loss_weight=0.5)))
    mt = build_model(ct, 7)
    gold["tap0_reco"] = trace_dict(generate_kv_recompute(mt, prompts[0], 0.99 / 64, 10))
    gold["tap0_pipe"] = trace_dict(generate_pipeline(partition(mt, 4), prompts[0], 0.99 / 64, 10))

    # ---- exit-head training KATs --------------------------------------------
    rng = np.random.default_rng(5)
    n, h, V = 24, 32, 96
    xh = rng.normal(size=(n, h))
    wh = rng.normal(0, 0.3, size=(V, h))
    nw = rng.normal(1.0, 0.1, size=h)
    tg = rng.integers(0, V, size=n)
    arrays.update(ce_x=xh, ce_w=wh, ce_norm=nw, ce_targets=tg)
    from eepipe.model import HeadDesc
    for kind in ("minimalistic", "norm+embed"):
        names = {"out": "out"}
        params = {"out": Tensor(wh.copy(), requires_grad=True)}
        if kind == "norm+embed":
            names["norm"] = "norm"
            params["norm"] = Tensor(nw.copy(), requires_grad=True)
        hd = HeadDesc("h", kind, 1, 1.0, False, names)
        xt = Tensor(xh.copy(), requires_grad=True)
        with Tape() as tape:
            logits = run_head(params, hd, xt, 4)
            loss = cross_entropy(logits, tg.reshape(n))
        grads = tape.backward(loss)
        tag = "min" if kind == "minimalistic" else "norm"
        arrays[f"ce_{tag}_logits"] = logits.data
        arrays[f"ce_{tag}_loss"] = np.array(loss.item())
        arrays[f"ce_{tag}_dx"] = grads[xt]
        arrays[f"ce_{tag}_dw"] = grads[params["out"]]
        if kind == "norm+embed":
            arrays["ce_norm_dnorm"] = grads[params["norm"]]

    # ---- weighted loss gradients (single-device oracle) ----------------------
    cw = ModelConfig(4, 32, 4, 64, 16, exits=(ExitSpec(1, loss_weight=0.25), ExitSpec(2, "norm+embed", 0.5)),
                     tie_embeddings=True)
    mw = build_model(cw, 3)
    batch = np.random.default_rng(9).integers(0, 64, size=(4, 13))
    arrays["wl_batch"] = batch
    grads, per_exit = single_device_gradients(mw, batch, [0.25, 0.5, 1.0], 2)
    gold["wl_per_exit"] = {k: float(v) for k, v in per_exit.items()}
    for name, g in grads.items():
        arrays[f"wl_grad::{name}"] = g

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    print("wrote", len(gold), "json keys,", len(arrays), "arrays")


if __name__ == "__main__":
    main()
