"""Profiling driver (run under ncu on the GPU box): full-depth decode passes
of the C3 7B model for one row, plus exit-head evaluations.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/prof_decode.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import MAX_DEFERRED, c3_config, prompt_tokens  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402


def main():
    passes = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 128  # first row's position
    cfg = c3_config()
    model = build_model(cfg, 0, init="device", dtype=torch.bfloat16)
    # builds the engine + one short generation (exercises heads)
    I.generate_kv_recompute(model, prompt_tokens(), 1.0, 2, MAX_DEFERRED)
    eng = next(iter(model.__dict__["_ee_engines"].values()))
    L = cfg.num_layers
    with torch.cuda.stream(eng.stream):
        eng.kv.reset()
        eng._grow(rows)
        eng.upload_ctrl([ctx + r for r in range(rows)])
        for _ in range(passes):
            eng.run_layers(0, L, rows, [rows] * L, ctx + rows, 0)
        eng.upload_ctrl(list(range(rows)))
        for i in range(passes):
            eng.eval_head(eng.heads[-1], eng.ctrl_ptr(0), rows, 1.0, i)
        eng.fetch_results(passes)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
