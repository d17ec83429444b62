"""Time the training attention at a config's layer shape: own tcgen05
kernels (ee_attn_train_fwd / _bwd) vs torch SDPA (cuDNN / flash), forward
and forward + backward, CUDA events, and TFLOP/s on the causal FLOP count
(fwd 2 matmuls x 2 B H S^2 dh / 2; bwd 2.5x fwd).

    python tools/time_attn_train.py [B S H]      (default C2: 2 2048 16)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2312_04916_b200.training import _AttnFn  # noqa: E402


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
    return a.elapsed_time(b) / reps


def main():
    B, S, H = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (2, 2048, 16)
    h = H * 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(B, S, h, device="cuda", generator=g).bfloat16().requires_grad_()
               for _ in range(3))
    do = torch.randn(B, S, h, device="cuda", generator=g).bfloat16()
    fwd_flop = 2 * 2 * B * H * S * S * 128 / 2
    F = torch.nn.functional
    split = lambda t: t.view(B, S, H, 128).transpose(1, 2)  # noqa: E731

    def own_f():
        return _AttnFn.get().apply(q, k, v, H)

    def own_fb():
        o = own_f()
        torch.autograd.backward(o, do)

    def sdpa_f():
        return F.scaled_dot_product_attention(split(q), split(k), split(v),
                                              is_causal=True).transpose(1, 2).reshape(B, S, h)

    def sdpa_fb():
        o = sdpa_f()
        torch.autograd.backward(o, do)

    for name, f, fb in (("own tcgen05", own_f, own_fb), ("torch SDPA", sdpa_f, sdpa_fb)):
        with torch.no_grad():
            tf = timeit(f)
        tfb = timeit(fb)
        print(f"{name:12s} B={B} S={S} H={H}: fwd {tf * 1e3:7.1f} us ({fwd_flop / tf / 1e9:6.0f} "
              f"TFLOP/s), fwd+bwd {tfb * 1e3:7.1f} us ({3.5 * fwd_flop / tfb / 1e9:6.0f} TFLOP/s)")


if __name__ == "__main__":
    main()
