"""Full-depth C3 decode pass time (1 row and 5 rows) vs context length, with
and without attention (EE_ABLATE=2 in a second process): how much of the
pass the attention costs as the context grows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402


def main():
    cfg = bench.c3_config()
    model = build_model(cfg, 0, init="device", dtype=torch.bfloat16)
    I.generate_kv_recompute(model, bench.prompt_tokens(), 1.0, 2, 4)
    eng = next(iter(model.__dict__["_ee_engines"].values()))
    L, st = cfg.num_layers, eng.stream
    with torch.cuda.stream(st):
        eng.kv.reset()
        eng._grow(16)
        for rows in [int(r) for r in os.environ.get('ROWS', '1,5').split(',')]:
            for ctx in [int(c) for c in os.environ.get('CTXS', '128,512,1024,2000').split(',')]:
                eng.upload_ctrl([ctx - rows + 1 + r for r in range(rows)])
                for _ in range(2):
                    eng.run_layers(0, L, rows, [rows] * L, ctx, 0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(10):
                    eng.run_layers(0, L, rows, [rows] * L, ctx, 0)
                b.record(st)
                st.synchronize()
                print(f"rows {rows} ctx {ctx}: {a.elapsed_time(b) / 10:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
