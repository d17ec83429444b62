"""Per-CTA start / end of the training attention kernels (trace build
libee_trace.so): busy time per CTA, sum over CTAs / 148 SMs vs the kernel
span, and the start-order histogram -- is a kernel bound by per-CTA work,
by prologue / epilogue, or by its schedule?

    python tools/attn_cta_timeline.py [B S H]      (default C2: 2 2048 16)
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402

lib = _lib.load(os.path.join(ROOT, "paper_2312_04916_b200", "libee_trace.so"))
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402

B, S, H = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2, 2048, 16)
h = H * 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(B * S, h, device="cuda", generator=g).bfloat16() for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(B, H, S, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
dsum = torch.empty_like(lse)
for _ in range(3):
    call("ee_attn_train_fwd", ptr(q), h, ptr(k), h, ptr(v), h, B, S, H, ptr(o), h, ptr(lse),
         stream_ptr())
    call("ee_attn_train_bwd", ptr(q), h, ptr(k), h, ptr(v), h, ptr(o), h, ptr(do), h, ptr(lse),
         B, S, H, ptr(dq), h, ptr(dk), h, ptr(dv), h, ptr(dsum), stream_ptr())
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 2048 * 4))()
lib.ee_trace_attn_cta(buf)
nt = S // 128
grids = {0: H * (nt // 2) * B, 1: H * nt * B, 2: H * nt * B}
for kname, kk in (("fwd", 0), ("bwd_kv", 1), ("bwd_q", 2)):
    n = grids[kk]
    st = [buf[(kk * 2048 + i) * 4] for i in range(n)]
    en = [buf[(kk * 2048 + i) * 4 + 1] for i in range(n)]
    f2 = [buf[(kk * 2048 + i) * 4 + 2] for i in range(n)]
    f3 = [buf[(kk * 2048 + i) * 4 + 3] for i in range(n)]
    t0 = min(st)
    span = (max(en) - t0) / 1e3
    busy = sum(e - s for s, e in zip(st, en)) / 1e3
    durs = sorted((e - s) / 1e3 for s, e in zip(st, en))
    late = sorted((s - t0) / 1e3 for s in st)
    print(f"{kname:7s} CTAs {n:4d} span {span:7.1f} us  busy/148 {busy / 148:7.1f} us  "
          f"CTA us min {durs[0]:.1f} med {durs[len(durs) // 2]:.1f} max {durs[-1]:.1f}  "
          f"last start {late[-1]:.1f} us")
    # per-y (work size) mean CTA duration
    ny = n // (H * B)
    per = []
    for y in range(ny):
        ids = [x + H * (y + ny * z) for z in range(B) for x in range(H)]
        per.append(sum((en[i] - st[i]) / 1e3 for i in ids) / len(ids))
    print("   mean us by blockIdx.y:", " ".join(f"{p:.1f}" for p in per))
    if any(f2):
        pro = sorted((a - s) / 1e3 for s, a in zip(st, f2))
        epi = sorted((e - a) / 1e3 for a, e in zip(f3, en))
        print(f"   prologue (start -> first S issued) med {pro[len(pro) // 2]:.2f} max {pro[-1]:.2f} us;"
              f" epilogue (last MMA done -> end) med {epi[len(epi) // 2]:.2f} max {epi[-1]:.2f} us")
