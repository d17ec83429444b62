"""Time the CTA-pair tcgen05 GEMM at the C2 backbone shapes (T = 8192 rows =
microbatch 4 x 2048): linear forward / dgrad (bf16 out), the GELU-fused MLP
up-projection, and the float32 weight-gradient accumulation; CUDA events,
TFLOP/s.  Run with EE_GEMM_STREAMK=0 for the plain round-robin schedule.

    python tools/time_gemm.py [T]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    _lib.load()
    h, f = 2048, 8192
    rnd = lambda *s: (torch.randn(*s, device="cuda") * 0.02).bfloat16()  # noqa: E731
    tag = "streamK" if os.environ.get("EE_GEMM_STREAMK", "1") != "0" else "plain"
    tot_us = tot_fl = 0.0
    for name, K, N in (("qkv", h, 3 * h), ("wo", h, h), ("w1", h, f), ("w2", f, h)):
        x, w = rnd(T, K), rnd(K, N)
        y = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
        dy = rnd(T, N)
        dx = torch.empty(T, K, device="cuda", dtype=torch.bfloat16)
        dw = torch.zeros(K, N, device="cuda")
        fl = 2.0 * T * K * N
        for kind, fn in (
                ("fwd", lambda: call("ee_linear_fwd", ptr(x), ptr(w), T, K, N, None, ptr(y), stream_ptr())),
                ("dgrad", lambda: call("ee_linear_dgrad", ptr(dy), ptr(w), T, K, N, None, ptr(dx),
                                       stream_ptr())),
                ("wgrad", lambda: call("ee_wgrad_accum", ptr(x), ptr(dy), T, K, N, ptr(dw), stream_ptr()))):
            us = timeit(fn)
            tot_us += us
            tot_fl += fl
            print(f"{tag:8s} {name:4s} {kind:6s} T={T} K={K:5d} N={N:5d}: {us:7.1f} us "
                  f"{fl / us / 1e6:7.0f} TFLOP/s")
    print(f"{tag:8s} total {tot_us:.1f} us, {tot_fl / tot_us / 1e6:.0f} TFLOP/s")


if __name__ == "__main__":
    main()
