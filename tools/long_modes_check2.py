"""Prompt-1024 consistency matrix on the 7B model: recompute (max_deferred 4
and 1), pipeline P=2 and P=4; prints which traces agree bitwise."""
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
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=n)]
    runs = {
        "reco4": I.generate_kv_recompute(model, prompt, 0.8, 8, 4),
        "reco1": I.generate_kv_recompute(model, prompt, 0.8, 8, 1),
        "pipe2": I.generate_pipeline(partition(model, 2, copy=False), prompt, 0.8, 8),
        "pipe4": I.generate_pipeline(partition(model, 4, copy=False), prompt, 0.8, 8),
    }
    keys = list(runs)
    for i, a in enumerate(keys):
        for b in keys[i + 1:]:
            print(a, b, runs[a].confidences == runs[b].confidences)
    print("reco4 conf[1]", runs["reco4"].confidences[1])
    print("pipe4 conf[1]", runs["pipe4"].confidences[1])


if __name__ == "__main__":
    main()
