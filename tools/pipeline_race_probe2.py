"""Pipeline-mode divergence probe: log, per stage and message, the rows'
checksum at every head check; compare two runs and print the first event
whose checksum differs (with the checksum of the same stage's INPUT rows)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402

LOG = []
_orig = I._InferStage._check_heads


def _check(self, msg, local, n):
    torch.cuda.current_stream().synchronize()
    x = self.eng.x[:n].double()
    LOG.append((self.spec.index, tuple(msg.positions)[:2], local, float(x.sum()), float((x * x).sum())))
    return _orig(self, msg, local, n)


I._InferStage._check_heads = _check


def main():
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=8)]
    part = partition(model, 2, copy=False)
    logs = []
    zero = os.environ.get("ZERO_KV") == "1"
    for run in range(4):
        LOG.clear()
        if zero:
            for spec in part.stages:
                for eng in spec.__dict__.get("_ee_engines", {}).values():
                    eng.kv.data.zero_()
            torch.cuda.synchronize()
        tr = I.generate_pipeline(part, prompt, float(os.environ.get("THR", "0.8")), 12)
        torch.cuda.synchronize()
        logs.append((sorted(LOG), tr.confidences))
    for run in range(1, 4):
        a, b = logs[0][0], logs[run][0]
        print(f"run {run}: trace equal {logs[run][1] == logs[0][1]}, events {len(a)} vs {len(b)}")
        for ea, eb in zip(a, b):
            if ea != eb:
                print("  first differing event:", ea, eb)
                break


if __name__ == "__main__":
    main()
