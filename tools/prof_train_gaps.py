"""GPU idle-gap census of one C2 training step (torch.profiler / CUPTI
kernel records): busy vs span and the kernel pairs around the largest idle
gaps (host launch / synchronisation bubbles)."""
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
        torch.cuda.synchronize()

    for _ in range(2):
        step()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        step()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    pairs, end, prev, gaps = {}, ev[0].time_range.end, ev[0], []
    for e in ev[1:]:
        g = e.time_range.start - end
        if g > 0:
            gaps.append(g)
            k = (prev.name[:45], e.name[:45])
            pairs.setdefault(k, [0, 0.0])
            pairs[k][0] += 1
            pairs[k][1] += g
        if e.time_range.end >= end:
            end, prev = e.time_range.end, e
    print(f"kernels={len(ev)} span={span/1e3:.1f} ms busy={busy/1e3:.1f} ms idle={(span-busy)/1e3:.1f} ms")
    for lo, hi in ((0, 5), (5, 20), (20, 100), (100, 1e9)):
        sel = [g for g in gaps if lo < g <= hi]
        print(f"  gaps ({lo}, {hi}] us: n={len(sel)} sum={sum(sel)/1e3:.1f} ms")
    for (a, b), (c, t) in sorted(pairs.items(), key=lambda x: -x[1][1])[:14]:
        print(f"  {c:5d}x {t/1e3:7.2f} ms  after {a!r} before {b!r}")
    t0 = ev[0].time_range.start
    end, prev = ev[0].time_range.end, ev[0]
    for e in ev[1:]:
        g = e.time_range.start - end
        if g > 1000:
            print(f"  big gap {g/1e3:.2f} ms at {(end - t0)/1e3:.1f} ms: after {prev.name[:50]!r} before {e.name[:50]!r}")
        if e.time_range.end >= end:
            end, prev = e.time_range.end, e




def cpu_table():
    """CPU self-time census of one step (python tools/prof_train_gaps.py cpu)."""
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
        torch.cuda.synchronize()

    for _ in range(2):
        step()
    with profile(activities=[ProfilerActivity.CPU], with_stack=True) as prof:
        step()
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
    seen = {}
    for e in prof.events():
        if e.name in ("cudaStreamSynchronize", "cudaEventSynchronize"):
            st = " <- ".join(f for f in (e.stack or [])[:6])
            key = (e.name, st)
            seen.setdefault(key, [0, 0.0])
            seen[key][0] += 1
            seen[key][1] += e.cpu_time_total
    for (n, st), (c, t) in sorted(seen.items(), key=lambda x: -x[1][1])[:8]:
        print(f"{n} x{c} {t/1e3:.1f} ms: {st}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "cpu":
        cpu_table()
    else:
        main()
