"""Localise pipeline-mode run-to-run differences on the 7B model: after two
identical generate_pipeline runs, compare every stage's KV cache position by
position and report the first (stage, layer, position) that differs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402


def snapshot(part, npos):
    out = []
    for spec in part.stages:
        eng = next(iter(spec.__dict__["_ee_engines"].values()))
        out.append(eng.kv.data[:, :, :npos].clone())
    return out


def main():
    n_prompt = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ntok = 16
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=n_prompt)]
    part = partition(model, P, copy=False)
    snaps, traces = [], []
    for run in range(4):
        tr = I.generate_pipeline(part, prompt, 0.8, ntok)
        torch.cuda.synchronize()
        traces.append(tr)
        snaps.append(snapshot(part, n_prompt + ntok))
    for run in range(1, 4):
        same = traces[run].confidences == traces[0].confidences
        print(f"run {run} vs 0: trace equal {same}")
        for s, (a, b) in enumerate(zip(snaps[0], snaps[run])):
            diff = (a != b)
            if diff.any():
                idx = diff.nonzero()
                first = idx[idx[:, 2].argmin()]
                print(f"  stage {s + 1}: first differing (layer slot, k/v, pos) = {first.tolist()}, "
                      f"positions differing: {sorted(set(idx[:, 2].tolist()))[:10]}")
                break


if __name__ == "__main__":
    main()
