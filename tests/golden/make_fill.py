"""Bubble-fill golden gradients from the REFERENCE executor (build container
only; `/root/reference` does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python python tests/golden/make_fill.py

The reference's own fill setup (tests/test_pipeline.py:258-266 of eepipe):
ModelConfig(8, 32, 4, 64, 16, exits at 2 (0.3) and 4 (0.6)), seed 17,
partition P=4, batch default_rng(18) 8x9, plan_bubble_fill(4, 0.5), fill rows
drawn next from the same generator.  Runs `run_iteration_1f1b` with and
without the plan (float64, numpy backend) and stores both gradient maps and
the per-exit losses in tests/golden/fill.npz / fill.json.
"""
import json
import os
import sys

import numpy as np

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from eepipe.bubblefill import plan_bubble_fill  # noqa: E402
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
    with open(os.path.join(HERE, "fill.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote fill.npz / fill.json:", meta["part1_depths"], meta["part2_bwd_depths"],
          meta["microbatches"])


if __name__ == "__main__":
    main()
