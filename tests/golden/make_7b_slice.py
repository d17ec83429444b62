"""Generate the 7B-WIDTH slice fixture from the REFERENCE implementation
(build container only).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python python tests/golden/make_7b_slice.py

ModelConfig(2, 4096, 32, 50304, 2048, exits=(1: minimalistic 0.1)) with the
reference's `build_model(cfg, 0)` (float64, ~8 GB host RAM), prompt
`default_rng(1).integers(0, 50304, 8)`, `generate_kv_recompute` at
threshold 1.0 (6 tokens, every head evaluated and logged) and at 0.05 (a
threshold inside the exit_l1 confidence spread, so early exits and deferred
recomputation happen at real width).  Writes tests/golden/golden_7b.json.
"""
import json
import os
import sys

import numpy as np

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from eepipe import kernels  # noqa: E402
from eepipe.inference import generate_kv_recompute  # noqa: E402
from eepipe.model import ExitSpec, ModelConfig, build_model  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, OUT)
from make_golden import params_digest, trace_dict  # noqa: E402


def main():
    cfg = ModelConfig(2, 4096, 32, 50304, 2048, exits=(ExitSpec(1, "minimalistic", 0.1),))
    m = build_model(cfg, 0)
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, 50304, size=8)]
    gold = {"backend": kernels.BACKEND, "prompt": prompt, "digest": params_digest(m)}
    gold["thr1"] = trace_dict(generate_kv_recompute(m, prompt, 1.0, 6))
    gold["thr005"] = trace_dict(generate_kv_recompute(m, prompt, 0.05, 6))
    with open(os.path.join(OUT, "golden_7b.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print(gold["thr1"]["tokens"], gold["thr005"]["exit_layers"])


if __name__ == "__main__":
    main()
