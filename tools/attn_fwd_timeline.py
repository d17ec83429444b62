"""Per-key-tile timeline of CTA 0 of the training attention forward (trace
build libee_trace.so): S issued / S seen by the softmax / P published / PV
issued, for tiles A and B, in us relative to the first S issue."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402

lib = _lib.load(os.path.join(ROOT, "paper_2312_04916_b200", "libee_trace.so"))
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402

B, S, H = 2, 2048, 16
h = H * 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B * S, h, device="cuda", generator=g).bfloat16() for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty(B, H, S, device="cuda")
for _ in range(3):
    call("ee_attn_train_fwd", ptr(q), h, ptr(k), h, ptr(v), h, B, S, H, ptr(o), h, ptr(lse),
         stream_ptr())
if len(sys.argv) > 1 and sys.argv[1] == "bwd":  # dK/dV kernel instead (events per q half)
    do = torch.randn_like(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    dsum = torch.empty_like(lse)
    for _ in range(2):
        call("ee_attn_train_bwd", ptr(q), h, ptr(k), h, ptr(v), h, ptr(o), h, ptr(do), h, ptr(lse),
             B, S, H, ptr(dq), h, ptr(dk), h, ptr(dv), h, ptr(dsum), stream_ptr())
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4 * 2 * 32))()
lib.ee_trace_attn_fwd(buf)
t = [[[buf[(e * 2 + tt) * 32 + j] for j in range(32)] for tt in range(2)] for e in range(4)]
t0 = t[0][0][0]
names = ["S issued", "PV/acc issued", "S seen", "P published"]
for tt in range(2):
    print("tile", "AB"[tt])
    for j in range(16):
        row = [(t[e][tt][j] - t0) / 1e3 if t[e][tt][j] else float("nan") for e in range(4)]
        print(f"  j={j:2d} " + "  ".join(f"{names[e]} {row[e]:7.2f}" for e in (0, 2, 3, 1)))
