"""Bubble-fill golden gradients from the REFERENCE executor (build container
only; `/root/reference` does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python python tests/golden/make_fill.py

The reference's own fill setup (tests/test_pipeline.py:258-266 of eepipe):
ModelConfig(8, 32, 4, 64, 16, exits at 2 (0.3) and 4 (0.6)), seed 17,
partition P=4, batch default_rng(18) 8x9, plan_bubble_fill(4, 0.5), fill rows
drawn next from the same generator.  Runs `run_iteration_1f1b` with and
without the plan (float64, numpy backend) and stores both gradient maps and
the per-exit losses in tests/golden/fill.npz / fill.json.  Also runs the
reference `train` with fill_bubbles on a 4-layer / 4-stage model (3 Adam
steps) and stores its per-step losses, microbatch counts and the regular and
fill batches its corpus served.
"""
import json
import os
import sys

import numpy as np

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from eepipe.bubblefill import plan_bubble_fill, truncated_part1_depths  # noqa: E402
from eepipe.config import RunConfig  # noqa: E402
from eepipe.training import train  # noqa: E402
from eepipe.model import ExitSpec, ModelConfig, build_model, partition  # noqa: E402
from eepipe.pipeline import IterationOptions, apply_fill, run_iteration_1f1b  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cfg = ModelConfig(8, 32, 4, 64, 16,
                      exits=(ExitSpec(2, loss_weight=0.3), ExitSpec(4, loss_weight=0.6)))
    model = build_model(cfg, 17)
    part = partition(model, 4)
    rng = np.random.default_rng(18)
    batch = rng.integers(0, 64, size=(8, 9))
    plan = plan_bubble_fill(4, 0.5)
    depths, _ = apply_fill(plan, part, 4)
    n_extra = sum(1 for d in depths if d is not None) + plan.k_part2
    fill_rows = rng.integers(0, 64, size=(2 * n_extra, 9))
    plain, rep_p = run_iteration_1f1b(part, batch, IterationOptions(microbatch_size=2))
    filled, rep_f = run_iteration_1f1b(part, batch, IterationOptions(
        microbatch_size=2, fill_plan=plan, fill_batch=fill_rows))
    arrays = {"batch": batch, "fill_rows": fill_rows}
    for n, g in plain.items():
        arrays["plain/" + n] = g
    for n, g in filled.items():
        arrays["filled/" + n] = g
    np.savez_compressed(os.path.join(HERE, "fill.npz"), **arrays)
    meta = {"config": [8, 32, 4, 64, 16], "exits": [[2, 0.3], [4, 0.6]], "seed": 17,
            "f_over_b": 0.5, "part1_depths": [d for d in depths],
            "part2_bwd_depths": list(plan.part2_bwd_depths),
            "microbatches": rep_f.microbatches,
            "plain_losses": rep_p.per_exit_losses, "filled_losses": rep_f.per_exit_losses}
    # train() with bubble filling (eepipe/training.py:64-136)
    tcfg = ModelConfig(4, 64, 4, 128, 64, exits=(ExitSpec(1, "minimalistic", 0.25),
                                                 ExitSpec(2, "minimalistic", 0.5)))
    rc = RunConfig(model=tcfg, stages=4, microbatch_size=2, global_batch_size=8, steps=3,
                   data_seq_len=32, learning_rate=3e-3, seed=0, fill_bubbles=True,
                   fill_f_over_b=0.5)
    _, hist = train(rc, rc.corpus())
    tplan = plan_bubble_fill(4, 0.5)
    tpart = partition(build_model(tcfg, 0), 4)
    tdepths = truncated_part1_depths(tplan, tpart.exit_stages())
    n_fill = sum(1 for d in tdepths if d is not None) + tplan.k_part2
    corpus = rc.corpus()
    arrays["train_batches"] = np.stack([corpus.batch(8, 33, st) for st in range(3)])
    arrays["train_fill_batches"] = np.stack([corpus.batch(n_fill * 2, 33, st + 10**9)
                                             for st in range(3)])
    meta["train"] = {"config": [4, 64, 4, 128, 64], "exits": [[1, 0.25], [2, 0.5]],
                     "stages": 4, "steps": 3, "lr": 3e-3, "f_over_b": 0.5,
                     "losses": [h["losses"] for h in hist],
                     "microbatches": [h["microbatches"] for h in hist]}
    np.savez_compressed(os.path.join(HERE, "fill.npz"), **arrays)
    with open(os.path.join(HERE, "fill.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote fill.npz / fill.json:", meta["part1_depths"], meta["part2_bwd_depths"],
          meta["microbatches"])


if __name__ == "__main__":
    main()
