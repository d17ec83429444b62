"""Generate the bf16-ROUNDED-WEIGHT fixtures from the REFERENCE implementation
(build container only; `/root/reference` does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python python tests/golden/make_bf16_golden.py [l2|l16|trained]

The bench path computes with bf16 weights.  To pin it to the reference, the
reference itself (float64 arithmetic, numpy backend) is run on the SAME
weights the GPU sees: every parameter of `build_model(cfg, 0)` (or of the
reference-trained checkpoint) rounded to bf16 (round-to-nearest-even, as the
device cast does) and widened back to float64.  What remains between the two
runs is the GPU's bf16 activations / KV cache and fp32 accumulation, so token
and exit-layer sequences must agree except where a decision sits within
tolerance of the threshold (or an argmax near-tie); tests/test_gpu_bf16_parity.py
and tools/bf16_parity_report.py check that and print every such mismatch.
Every call of the reference's `exit_decision` is also recorded with its
top-5 (token, probability), so a flipped greedy token can be checked to be an
argmax near-tie of the REFERENCE's own distribution.

  l2      ModelConfig(2, 4096, 32, 50304, 2048, exit 1 minimalistic) — SURVEY
          B.3 slice; 2 prompts x thresholds {1.0, 0.3, 0.1, 0.05} x 12 tokens
          (KV recompute, max_deferred 4) + pipeline P=2 at 0.1
          -> tests/golden/golden_7b_bf16.json
  l16     ModelConfig(16, 4096, 32, 50304, 2048, exit 8 minimalistic) — the
          exit tap of C3 at real depth; 1 prompt x {1.0, 0.9, 0.8, 0.5, 0.3}
          x 8 tokens -> tests/golden/golden_7b16_bf16.json (used by
          tools/bf16_parity_report.py: the host float64 build takes minutes)
  trained the reference-trained C1-style checkpoint (tests/golden/trained_tiny.ckpt)
          rounded to bf16; its 3 prompts x {0.9, 0.8, 0.5} x 24 tokens, KV
          recompute (max_deferred 4) and pipeline P=2 -> tests/golden/trained_bf16.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import eepipe.inference as _inf  # noqa: E402
from eepipe import kernels  # noqa: E402
from eepipe.checkpoint import load_model  # noqa: E402
from eepipe.inference import generate_kv_recompute, generate_pipeline  # noqa: E402
from eepipe.model import ExitSpec, ModelConfig, build_model, partition  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, OUT)
from make_golden import params_digest, trace_dict  # noqa: E402


_DECISIONS = []
_exit_decision = _inf.exit_decision


def _recording_exit_decision(logits, threshold):
    """The reference's own exit_decision, unchanged, plus a record of the
    top-5 (token, probability) of every call: lets the GPU test prove that a
    flipped greedy token was an argmax near-tie in the REFERENCE's
    distribution (our token within tolerance of the reference's maximum)."""
    out = _exit_decision(logits, threshold)
    z = np.asarray(logits, dtype=np.float64)
    p = np.exp(z - z.max())
    p /= p.sum()
    top = np.argsort(-p, kind="stable")[:5]
    _DECISIONS.append({"token": int(out[1]), "conf": float(out[2]),
                       "top5": [[int(t), float(p[t])] for t in top]})
    return out


_inf.exit_decision = _recording_exit_decision


def traced(fn, *a):
    _DECISIONS.clear()
    d = trace_dict(fn(*a))
    d["decisions"] = list(_DECISIONS)
    return d


def round_bf16(model):
    """Every parameter -> bf16 (RNE) -> float64, in place."""
    for p in model.params.values():
        p.data[...] = torch.from_numpy(p.data).to(torch.bfloat16).double().numpy()


def slice_fixture(L, tap, prompts, thresholds, new, pipe_thr, name):
    cfg = ModelConfig(L, 4096, 32, 50304, 2048, exits=(ExitSpec(tap, "minimalistic", 0.1),))
    t0 = time.time()
    m = build_model(cfg, 0)
    round_bf16(m)
    print(f"built + rounded L={L} in {time.time() - t0:.0f} s", flush=True)
    gold = {"backend": kernels.BACKEND, "config": [L, 4096, 32, 50304, 2048, tap],
            "digest_bf16_rounded": params_digest(m), "prompts": prompts, "new_tokens": new,
            "runs": []}
    for pi, prompt in enumerate(prompts):
        for thr in thresholds:
            t0 = time.time()
            tr = traced(generate_kv_recompute, m, prompt, thr, new, 4)
            gold["runs"].append({"prompt": pi, "threshold": thr, "mode": "recompute",
                                 "max_deferred": 4, **tr})
            print(f"  prompt {pi} thr {thr}: {tr['tokens']} exits {tr['exit_layers']} "
                  f"({time.time() - t0:.0f} s)", flush=True)
        if pipe_thr is not None:
            tr = traced(generate_pipeline, partition(m, 2), prompt, pipe_thr, new)
            gold["runs"].append({"prompt": pi, "threshold": pipe_thr, "mode": "pipeline",
                                 "stages": 2, **tr})
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)


def trained_fixture():
    m = load_model(os.path.join(OUT, "trained_tiny.ckpt"))
    round_bf16(m)
    with open(os.path.join(OUT, "trained.json")) as f:
        prompts = json.load(f)["prompts"]
    gold = {"backend": kernels.BACKEND, "digest_bf16_rounded": params_digest(m),
            "prompts": prompts, "new_tokens": 24, "runs": []}
    part = partition(m, 2)
    for pi, prompt in enumerate(prompts):
        for thr in (0.9, 0.8, 0.5):
            tr = traced(generate_kv_recompute, m, prompt, thr, 24, 4)
            gold["runs"].append({"prompt": pi, "threshold": thr, "mode": "recompute",
                                 "max_deferred": 4, **tr})
            tr = traced(generate_pipeline, part, prompt, thr, 24)
            gold["runs"].append({"prompt": pi, "threshold": thr, "mode": "pipeline",
                                 "stages": 2, **tr})
    with open(os.path.join(OUT, "trained_bf16.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)


def main():
    which = sys.argv[1:] or ["trained", "l2", "l16"]
    p1 = [int(t) for t in np.random.default_rng(1).integers(0, 50304, size=8)]
    p2 = [int(t) for t in np.random.default_rng(2).integers(0, 50304, size=20)]
    if "trained" in which:
        trained_fixture()
    if "l2" in which:
        slice_fixture(2, 1, [p1, p2], (1.0, 0.3, 0.1, 0.05), 12, 0.1, "golden_7b_bf16.json")
    if "l16" in which:
        slice_fixture(16, 8, [p1], (1.0, 0.9, 0.8, 0.5, 0.3), 8, None, "golden_7b16_bf16.json")


if __name__ == "__main__":
    main()
