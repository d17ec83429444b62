"""CPU enqueue time vs GPU time of one C2 microbatch forward and backward
(is the training step launch-bound?)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import time_train_step as T  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402
from paper_2312_04916_b200.pipeline import StageCompute  # noqa: E402


def main():
    cfg = T.c2_config()
    master = build_model(cfg, 0, init="device", dtype=torch.float32)
    part = partition(master, 1, copy=False)
    heads = sorted(master.heads, key=lambda hd: (hd.layer_index, hd.is_final))
    w = {hd.key: hd.loss_weight for hd in heads}
    comp = StageCompute(part.stages[0], cfg, master, w, "cuda:0", None, torch.float32)
    rows = np.random.default_rng(0).integers(0, cfg.vocab_size, size=(2, 2049))
    tok, tgt = rows[:, :-1], rows[:, 1:]
    for it in range(4):
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        c0 = time.perf_counter()
        _, st = comp.forward(tok, tgt)
        c1 = time.perf_counter()
        e1.record()
        comp.backward(st, None)
        c2 = time.perf_counter()
        e2.record()
        torch.cuda.synchronize()
        c3 = time.perf_counter()
        print(f"fwd: cpu {1e3*(c1-c0):.1f} ms gpu {e0.elapsed_time(e1):.1f} ms | "
              f"bwd: cpu {1e3*(c2-c1):.1f} ms gpu {e1.elapsed_time(e2):.1f} ms | wall {1e3*(c3-c0):.1f}")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def fwd_cpu_table():
    from torch.profiler import ProfilerActivity, profile
    cfg = T.c2_config()
    master = build_model(cfg, 0, init="device", dtype=torch.float32)
    part = partition(master, 1, copy=False)
    heads = sorted(master.heads, key=lambda hd: (hd.layer_index, hd.is_final))
    w = {hd.key: hd.loss_weight for hd in heads}
    comp = StageCompute(part.stages[0], cfg, master, w, "cuda:0", None, torch.float32)
    rows = np.random.default_rng(0).integers(0, cfg.vocab_size, size=(2, 2049))
    tok, tgt = rows[:, :-1], rows[:, 1:]
    for _ in range(2):
        _, st = comp.forward(tok, tgt)
        comp.backward(st, None)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU]) as prof:
        _, st = comp.forward(tok, tgt)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=22))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "fwd":
    fwd_cpu_table()
