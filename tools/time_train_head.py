"""Time the fused training exit head at the C2 shape (n=4096 = 2 x 2048
tokens, h=2048, V=50304) with CUDA events; TFLOP/s on the algorithmic
6 n h V."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2312_04916_b200.training import exit_head_loss_and_grads  # noqa: E402


def main():
    n, h, V = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 2048, 50304)))
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, h, device="cuda", generator=g).bfloat16()
    w = (torch.randn(V, h, device="cuda", generator=g) * 0.02).bfloat16()
    t = torch.randint(0, V, (n,), device="cuda", generator=g)
    acc = torch.zeros(V, h, device="cuda")
    for _ in range(2):
        exit_head_loss_and_grads(x, w, t, 1.0, dw_acc=acc)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        loss, dx, _ = exit_head_loss_and_grads(x, w, t, 1.0, dw_acc=acc)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    tf = 6 * n * h * V / (ms * 1e-3) / 1e12
    print(f"n={n} h={h} V={V}: {ms:.3f} ms/head  {tf:.1f} TFLOP/s (6nhV)  loss={float(loss):.5f}")


if __name__ == "__main__":
    main()
