"""Kernel-time census (torch.profiler / CUPTI) of one C2 training step:
per-kernel time, the step's span, and the span's GPU-idle share (no kernel
of either stream running).

    python tools/prof_train_step.py [M mb]      (default 4 4, as bench.py)
"""
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
    M, mb = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (4, 4)
    seq = 2048
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
    busy, cur_s, cur_e = 0.0, None, None
    for e in ev:  # union of kernel intervals
        a, b = e.time_range.start, e.time_range.end
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    busy += cur_e - cur_s
    print(f"M={M} mb={mb}: span {span/1e3:.1f} ms, kernel time {tot/1e3:.1f} ms, {len(ev)} kernels, "
          f"GPU idle {100 * (1 - busy / span):.1f}% of the span")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{t/1e3:8.2f} ms {100*t/tot:5.1f}% {c:6d}  {k}")


if __name__ == "__main__":
    main()
