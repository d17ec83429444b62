"""Generate the TRAINED fixture from the REFERENCE implementation (run in the
build container only; `/root/reference` does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python \
        python tests/golden/make_trained.py

SURVEY Appendix B.2 at reduced width (so the checkpoint stays ~2 MB in git):
the reference's own `train` (eepipe/training.py:64-136; Adam, lr 3e-3, 2
pipeline stages, microbatch 2, global batch 8, MarkovCorpus seed 0, 300
steps) on ModelConfig(4, 64, 4, 128, 64, exits 1:0.25, 2:0.5), saved with the
reference's `save_model` (eepipe/checkpoint.py:79-100) as
`tests/golden/trained_tiny.ckpt`.  Random-init confidences at this width sit
near 1/V, so only a trained model exercises early exits at thresholds 0.8 /
0.9; this one exits early on a mix of tokens (tests/test_checkpoint.py,
tests/test_gpu_trained.py).

`trained.json` holds: the training loss history, KV-recompute traces for 3
corpus prompts x thresholds {1.0, 0.9, 0.8, 0.5} x max_deferred {1, 4} and
pipeline (P=2) traces, plus a fresh 3-step Adam run (per-step losses) and
`trained.npz` the parameters after those 3 steps for a few tensors (the
optimizer-step parity anchor, eepipe/training.py:33-53).
"""

import json
import os
import sys

import numpy as np

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from eepipe import kernels  # noqa: E402
from eepipe.checkpoint import save_model  # noqa: E402
from eepipe.config import RunConfig  # noqa: E402
from eepipe.inference import generate_kv_recompute, generate_pipeline  # noqa: E402
from eepipe.model import ExitSpec, ModelConfig, build_model, partition  # noqa: E402
from eepipe.training import train  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, OUT)
from make_golden import params_digest, trace_dict  # noqa: E402

KEEP = ("tok_emb", "layer1.wq", "layer2.w1", "final.out", "exit_l1.out", "final.norm",
        "layer3.mlp_norm")


def main():
    cfg = ModelConfig(4, 64, 4, 128, 64, exits=(ExitSpec(1, "minimalistic", 0.25),
                                                ExitSpec(2, "minimalistic", 0.5)))
    rc = RunConfig(model=cfg, stages=2, microbatch_size=2, global_batch_size=8, steps=300,
                   data_seq_len=32, learning_rate=3e-3, seed=0)
    corpus = rc.corpus()
    model, hist = train(rc, corpus)
    save_model(os.path.join(OUT, "trained_tiny.ckpt"), model)
    gold = {"backend": kernels.BACKEND, "digest": params_digest(model),
            "train": {"stages": 2, "microbatch_size": 2, "global_batch_size": 8, "steps": 300,
                      "data_seq_len": 32, "learning_rate": 3e-3, "seed": 0, "optimizer": "adam"},
            "loss_history": [h["losses"] for h in hist]}
    prompts = [[int(v) for v in corpus.batch(1, 8, 10**6 + i)[0]] for i in range(3)]
    gold["prompts"] = prompts
    runs = []
    part = partition(model, 2)
    for pi, prompt in enumerate(prompts):
        for thr in (1.0, 0.9, 0.8, 0.5):
            for md in (1, 4):
                runs.append({"prompt": pi, "threshold": thr, "max_deferred": md,
                             "recompute": trace_dict(generate_kv_recompute(model, prompt, thr, 24, md))})
            runs.append({"prompt": pi, "threshold": thr,
                         "pipeline": trace_dict(generate_pipeline(part, prompt, thr, 24))})
    gold["runs"] = runs

    # fresh 3-step Adam run from the same seed: per-step losses + parameters
    rc3 = RunConfig(model=cfg, stages=2, microbatch_size=2, global_batch_size=8, steps=3,
                    data_seq_len=32, learning_rate=3e-3, seed=0)
    m3, h3 = train(rc3, rc3.corpus())
    gold["adam3_losses"] = [h["losses"] for h in h3]
    gold["adam3_digest"] = params_digest(m3)
    gold["init_digest"] = params_digest(build_model(cfg, 0))
    arrays = {f"adam3::{k}": m3.params[k].data for k in KEEP}
    arrays["adam3_batches"] = np.stack([rc3.corpus().batch(8, 33, s) for s in range(3)])

    with open(os.path.join(OUT, "trained.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "trained.npz"), **arrays)
    print("wrote trained fixture:", len(runs), "runs")


if __name__ == "__main__":
    main()
