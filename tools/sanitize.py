"""Small end-to-end run of every kernel family for compute-sanitizer:
tiled bf16 decode (KV recompute + pipeline, prefill GEMM, attention, heads),
fp32 parity decode, fused train head, RMSNorm, optimizer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition  # noqa: E402
from paper_2312_04916_b200.training import (Adam, exit_head_loss_and_grads, rmsnorm)  # noqa: E402


def main():
    cfg = ModelConfig(2, 512, 4, 256, 64, exits=(ExitSpec(1, "minimalistic", 0.3),))
    m = build_model(cfg, 1, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, 256, size=20)]
    I.generate_kv_recompute(m, prompt, 1.2 / 256, 6, 2)
    I.generate_pipeline(partition(m, 2, copy=False), prompt, 1.2 / 256, 6)
    small = build_model(ModelConfig(4, 32, 4, 64, 32, exits=(ExitSpec(2, loss_weight=0.5),)), 3)
    I.generate_kv_recompute(small, [1, 2, 3], 0.99 / 64, 5, 2, dtype="fp32")
    x = torch.randn(136, 256, device="cuda").bfloat16()
    w = (torch.randn(520, 256, device="cuda") * 0.05).bfloat16()
    t = torch.randint(0, 520, (136,), device="cuda")
    exit_head_loss_and_grads(x, w, t)
    xr = torch.randn(37, 264, device="cuda").bfloat16().requires_grad_()
    wr = torch.ones(264, device="cuda", requires_grad=True)
    rmsnorm(xr, wr).sum().backward()
    p = {"a": torch.zeros(1003, device="cuda")}
    Adam(1e-3).step(p, {"a": torch.ones(1003, device="cuda")}, 0.5)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
