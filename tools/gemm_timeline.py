"""Per-cluster unit timeline of the CTA-pair GEMM (trace build
libee_trace.so): for each cluster's units (tile, k-range, role) the MMA
start / end-of-issue and the epilogue start / end in us from the kernel's
first MMA; a linear forward of shape T x K -> N.

    python tools/gemm_timeline.py [T K N]       (default 8192 2048 2048)
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

T, K, N = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 2048, 2048)
x = (torch.randn(T, K, device="cuda") * 0.02).bfloat16()
w = (torch.randn(K, N, device="cuda") * 0.02).bfloat16()
y = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    call("ee_linear_fwd", ptr(x), ptr(w), T, K, N, None, ptr(y), stream_ptr())
torch.cuda.synchronize()
tl = (ctypes.c_ulonglong * (80 * 12 * 4))()
un = (ctypes.c_int * (80 * 12 * 4))()
lib.ee_trace_gemm(tl, un)
t0 = min(v for v in tl if v)
roles = "WwO"
ends = []
for c in list(range(0, 6)) + list(range(68, 74)):
    parts = []
    for j in range(12):
        b = (c * 12 + j) * 4
        if tl[b] == 0 or tl[b] < t0:
            continue
        t, k0, k1, r = un[b:b + 4]
        e = [(tl[b + i] - t0) / 1e3 if tl[b + i] >= t0 else float("nan") for i in range(4)]
        parts.append(f"[t{t} {k0}-{k1} {'whole writer owner'.split()[r][0]}: "
                     f"mma {e[0]:.1f}-{e[1]:.1f} epi {e[2]:.1f}-{e[3]:.1f}]")
    print(f"cl{c:2d} " + " ".join(parts))
for c in range(80):
    last = [tl[(c * 12 + j) * 4 + 3] for j in range(12) if tl[(c * 12 + j) * 4 + 3] >= t0]
    if last:
        ends.append((max(last) - t0) / 1e3)
print(f"cluster end us: min {min(ends):.1f} median {sorted(ends)[len(ends) // 2]:.1f} max {max(ends):.1f}")
