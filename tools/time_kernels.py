"""Per-kernel timing in steady state (warm L2 where it would be warm in a
real decode), CUDA events around N back-to-back launches of one ABI call.

    python tools/time_kernels.py        # EE_PDL=0 to disable PDL
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    lib = _lib.load()
    h, nh, V, smax = 4096, 32, 50304, 2048
    dev = "cuda:0"
    s = stream_ptr()
    x = torch.randn(16, h, device=dev)
    nw = torch.ones(h, device=dev)
    xn = torch.empty(16, 4 * h, dtype=torch.bfloat16, device=dev)
    res = {}
    res["rmsnorm m=1"] = timed(lambda: call("ee_rmsnorm_rows", ptr(x), h, None, 1, h, ptr(nw), 1e-6,
                                            ptr(xn), _lib.EE_BF16, s))
    kc = torch.randn(smax, h, device=dev).bfloat16()
    vc = torch.randn(smax, h, device=dev).bfloat16()
    q = torch.randn(16, h, device=dev)
    out = torch.empty(16, h, dtype=torch.bfloat16, device=dev)
    for ctx in (128, 320, 1024, 2047):
        for m in (1, 5):
            pos = torch.tensor([ctx - m + 1 + i for i in range(m)], dtype=torch.int32, device=dev)
            res[f"attention m={m} ctx={ctx}"] = timed(lambda: call(
                "ee_decode_attention", ptr(q), m, ptr(pos), ctx, ptr(kc), ptr(vc), nh, h // nh,
                _lib.EE_BF16, ptr(out), None, 0, s))
    # tiled GEMVs (random weights; rotate 4 copies so L2 never holds them)
    for name, N, K in (("qkv", 3 * h, h), ("wo", h, h), ("w1", 4 * h, h), ("w2", h, 4 * h),
                       ("head", V, h)):
        Ws = []
        for _ in range(4):
            w = torch.randn(N, K, device=dev).bfloat16()
            t = torch.empty(lib.ee_tiled_weight_bytes(N, K) // 2, dtype=torch.bfloat16, device=dev)
            call("ee_pack_tiled", ptr(w), N, K, ptr(t), s)
            Ws.append(t)
            del w
        xin = torch.randn(16, K, device=dev).bfloat16()
        o = torch.zeros(16, N, device=dev)
        for m in (1, 5):
            it = [0]

            def run():
                it[0] += 1
                call("ee_gemv", ptr(xin), m, K, ptr(Ws[it[0] & 3]), N, _lib.EE_BF16_TILED,
                     _lib.EE_EPI_STORE, ptr(o), N, s)
            us = timed(run)
            res[f"gemv_tiled {name} m={m}"] = us
            res[f"gemv_tiled {name} m={m} GB/s"] = N * K * 2 / (us * 1e-6) / 1e9
        del Ws
    for k, v in res.items():
        print(f"{k:32s} {v:10.2f}")


if __name__ == "__main__":
    main()
