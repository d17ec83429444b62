"""Standalone timing of the training RMSNorm forward / backward (with the
residual gradient) at a C2 microbatch shape (rows x h), CUDA events."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402


def main():
    n, h = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (8192, 2048)
    lib = _lib.load()
    x = torch.randn(n, h, device="cuda").bfloat16()
    g = torch.randn(n, h, device="cuda").bfloat16()
    r = torch.randn(n, h, device="cuda").bfloat16()
    w = torch.ones(h, device="cuda")
    y, gx = torch.empty_like(x), torch.empty_like(x)
    inv = torch.empty(n, device="cuda")
    gw = torch.empty(h, device="cuda")
    ws = torch.empty(lib.ee_workspace_bytes(_lib.EE_OP_RMSNORM_BWD, n, h, 0, 0, 0),
                     dtype=torch.uint8, device="cuda")
    import ctypes
    fwd = lambda: call("ee_rmsnorm_fwd", ptr(x), n, h, ptr(w), ctypes.c_float(1e-6), ptr(y),  # noqa: E731
                       ptr(inv), stream_ptr())
    bwd = lambda: call("ee_rmsnorm_bwd", ptr(x), ptr(w), ptr(inv), ptr(g), ptr(r), n, h,  # noqa: E731
                       ptr(gx), ptr(gw), 0, ptr(ws), ws.numel(), stream_ptr())
    for name, f, nbytes in (("fwd", fwd, 2 * n * h * 2), ("bwd+res", bwd, 4 * n * h * 2)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        print(f"{name}: {us:.1f} us, {nbytes / us / 1e3:.0f} GB/s ({n} x {h})")


if __name__ == "__main__":
    main()
