"""Run-to-run determinism of both decoding modes on the 7B model."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402


def main():
    n_prompt = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=n_prompt)]
    part = partition(model, P, copy=False)
    r = [I.generate_kv_recompute(model, prompt, 0.8, 16) for _ in range(3)]
    p = [I.generate_pipeline(part, prompt, 0.8, 16) for _ in range(3)]
    print("recompute runs equal:", all(x.confidences == r[0].confidences for x in r))
    print("pipeline runs equal:", all(x.confidences == p[0].confidences for x in p))
    print("modes equal:", r[0].confidences == p[0].confidences)
    for i, (a, b) in enumerate(zip(r[0].confidences, r[1].confidences)):
        if a != b:
            print("recompute run diff at", i, a, b)
            break
    for i, (a, b) in enumerate(zip(p[0].confidences, p[1].confidences)):
        if a != b:
            print("pipeline run diff at", i, a, b)
            break


if __name__ == "__main__":
    main()
