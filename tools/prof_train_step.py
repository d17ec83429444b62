"""Kernel-time census (torch.profiler / CUPTI) of one C2 training step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import time_train_step as T  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402
from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b  # noqa: E402
from paper_2312_04916_b200.training import Adam, apply_update  # noqa: E402


def main():
    M, mb, seq = 8, 2, 2048
    cfg = T.c2_config()
    master = build_model(cfg, 0, init="device", dtype=torch.float32)
    opt = Adam(3e-4)
    batch = np.random.default_rng(0).integers(0, cfg.vocab_size, size=(M * mb, seq + 1))

    part = partition(master, 1, copy=False)
    computes = []

    def step():
        grads, _ = run_iteration_1f1b(part, batch, IterationOptions(microbatch_size=mb),
                                      model=master, master_dtype=torch.float32,
                                      stage_computes=computes)
        apply_update(opt, master, grads, computes, 1.0 / M)

    step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    span = ev[-1].time_range.end - ev[0].time_range.start
    agg = {}
    for e in ev:
        k = e.name[:90]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    tot = sum(v[1] for v in agg.values())
    print(f"span {span/1e3:.1f} ms, kernel time {tot/1e3:.1f} ms, {len(ev)} kernels")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{t/1e3:8.2f} ms {100*t/tot:5.1f}% {c:6d}  {k}")


if __name__ == "__main__":
    main()
