"""Timeline of one decode layer (QKV GEMV -> attention -> wo -> w1 -> w2) from
%globaltimer probes in the profiling build libee_trace.so (-DEE_TRACE; build
with `python -m paper_2312_04916_b200.build_lib --trace`).  Prints, per
context length and row count, the median over repeats of each probe relative
to the QKV GEMV's first CTA entry (us)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402

lib = _lib.load(os.path.join(ROOT, "paper_2312_04916_b200", "libee_trace.so"))
import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402

NAMES_G = {0: "qkv entry", 2: "qkv post-wait", 1: "qkv exit", 4: "wo entry", 6: "wo post-wait",
           5: "wo exit", 8: "w1 entry", 10: "w1 post-wait", 9: "w1 exit", 12: "w2 entry",
           14: "w2 post-wait", 13: "w2 exit"}
NAMES_A = {0: "attn entry", 2: "attn post-wait first", 3: "attn post-wait last",
           11: "attn slab0 scores last", 13: "attn slab0 softmax last", 15: "attn slab0 PV last",
           1: "attn cluster barrier last",
           5: "attn K/V loaded last", 7: "attn block merge done last", 9: "attn chunk merge last"}


def read(fn):
    buf = (ctypes.c_ulonglong * 16)()
    fn(buf, 1)
    return list(buf)


def main():
    cfg = bench.c3_config()
    model = build_model(cfg, 0, init="device", dtype=torch.bfloat16)
    I.generate_kv_recompute(model, bench.prompt_tokens(), 1.0, 2, 4)
    eng = next(iter(model.__dict__["_ee_engines"].values()))
    st = eng.stream
    reps = int(os.environ.get("REPS", "20"))
    with torch.cuda.stream(st):
        eng.kv.reset()
        eng._grow(16)
        for rows in [int(r) for r in os.environ.get("ROWS", "1,5").split(",")]:
            for ctx in [int(c) for c in os.environ.get("CTXS", "192,2000").split(",")]:
                eng.upload_ctrl([ctx - rows + 1 + r for r in range(rows)])
                eng.run_layers(0, 2, rows, [rows] * 2, ctx, 0)
                st.synchronize()
                read(lib.ee_trace_gemv), read(lib.ee_trace_attention)
                samples = []
                for _ in range(reps):
                    eng.run_layers(4, 5, rows, [rows], ctx, 0)
                    st.synchronize()
                    g, a = read(lib.ee_trace_gemv), read(lib.ee_trace_attention)
                    t0 = g[0]
                    ev = {NAMES_G[i]: (g[i] - t0) / 1e3 for i in NAMES_G}
                    ev.update({NAMES_A[i]: (a[i] - t0) / 1e3 for i in NAMES_A
                               if a[i] not in (0, 2**64 - 1)})
                    samples.append(ev)
                keys = sorted(samples[0], key=lambda k: np.median([s[k] for s in samples]))
                print(f"rows {rows} ctx {ctx}:")
                for k in keys:
                    print(f"  {np.median([s[k] for s in samples]):8.2f} us  {k}")


if __name__ == "__main__":
    main()
