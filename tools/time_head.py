"""Steady-state timing of the fused inference exit head (ee_exit_head_infer,
tiled bf16, h=4096, V=50304) for m = 1, 5, 16 rows; 4 rotating weight copies
so L2 never holds the matrix."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_04916_b200 import _lib  # noqa: E402
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402


def main():
    lib = _lib.load()
    h, V = 4096, 50304
    s = stream_ptr()
    Ws = []
    for i in range(4):
        w = (torch.randn(V, h, device="cuda") * 0.02).bfloat16()
        t = torch.empty(lib.ee_tiled_weight_bytes(V, h) // 2, dtype=torch.bfloat16, device="cuda")
        call("ee_pack_tiled", ptr(w), V, h, None, ptr(t), s)
        Ws.append(t)
        del w
    ws = torch.zeros(lib.ee_workspace_bytes(_lib.EE_OP_EXIT_HEAD, 16, h, V, 0, 0), dtype=torch.uint8,
                     device="cuda")
    x = torch.randn(16, h, device="cuda")
    tok = torch.zeros(16, dtype=torch.int32, device="cuda")
    conf = torch.zeros(16, device="cuda")
    fire = torch.zeros(16, dtype=torch.uint8, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    for m in (1, 5, 16):
        it = [0]

        def run():
            it[0] += 1
            call("ee_exit_head_infer", ptr(x), h, None, m, h, None, ctypes.c_float(1e-6),
                 ptr(Ws[it[0] & 3]), V, _lib.EE_BF16_TILED, ctypes.c_float(0.5), ptr(tok),
                 ptr(conf), ptr(fire), ptr(bad), None, ptr(ws), ws.numel(), s)
        for _ in range(5):
            run()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(40):
            run()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 40 * 1e3
        print(f"exit head m={m:2d}: {us:7.1f} us  {V * h * 2 / us / 1e3:6.0f} GB/s")


if __name__ == "__main__":
    main()
