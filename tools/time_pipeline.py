"""C3 (7B) pipeline-based early-exit inference (`generate_pipeline`) with P
stage workers (threads + CUDA streams) on ONE GPU: tokens/s per threshold."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = bench.prompt_tokens()
    for P in (2, 4):
        part = partition(model, P, copy=False)
        I.generate_pipeline(part, prompt, 0.8, 4)
        for thr in (1.0, 0.8, 0.2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            tr = I.generate_pipeline(part, prompt, thr, n)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            print(f"P={P} thr={thr}: {len(tr.tokens) / dt:7.1f} tok/s  mean exit {tr.mean_exit_layer:5.2f}"
                  f"  modeled speedup {tr.speedup:.2f}")
    t = time.perf_counter()
    tr = I.generate_kv_recompute(model, prompt, 0.8, n)
    torch.cuda.synchronize()
    print(f"recompute thr=0.8: {len(tr.tokens) / (time.perf_counter() - t):7.1f} tok/s")


if __name__ == "__main__":
    main()
