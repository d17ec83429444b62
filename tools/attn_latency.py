"""Latency of the decode attention kernel alone (warm L2), serialised
launches (run with EE_PDL=0), against a trivial one-row kernel as the launch
floor.  python tools/attn_latency.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    lib = _lib.load()
    h, nh, smax = 4096, 32, 2048
    dev = "cuda:0"
    s = stream_ptr()
    x = torch.randn(16, h, device=dev)
    xb = torch.empty(16, h, dtype=torch.bfloat16, device=dev)
    ssq = torch.empty(16, h // 16, device=dev)
    print("row_stats m=1 (floor) %.2f us" % timed(
        lambda: call("ee_row_stats", ptr(x), h, 1, h, ptr(xb), ptr(ssq), s)))
    kc = torch.randn(smax, h, device=dev).bfloat16()
    vc = torch.randn(smax, h, device=dev).bfloat16()
    q = torch.randn(16, h, device=dev)
    out = torch.empty(16, h, dtype=torch.bfloat16, device=dev)
    wsb = lib.ee_workspace_bytes(_lib.EE_OP_ATTENTION, 16, h, 0, nh, smax)
    ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
    for ctx in (32, 192, 320, 640, 1024, 2000):
        for m in (1, 5, 16):
            pos = torch.tensor([ctx - m + 1 + i for i in range(m)], dtype=torch.int32, device=dev)
            us = timed(lambda: call("ee_decode_attention", ptr(q), m, ptr(pos), ctx, ptr(kc),
                                    ptr(vc), nh, h // nh, _lib.EE_BF16, ptr(out), ptr(ws),
                                    wsb, s))
            print(f"attention m={m} ctx={ctx}: {us:.2f} us", flush=True)


if __name__ == "__main__":
    main()
