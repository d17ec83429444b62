"""Small end-to-end run of every kernel family for compute-sanitizer:
tiled bf16 decode (KV recompute + pipeline, prefill GEMM, attention, heads),
fp32 parity decode, fused train head, RMSNorm, optimizer, fused-GELU MLP
GEMMs, weight-gradient accumulation, multi-row long-context attention
(cluster slab kernel), training attention fwd / bwd, backbone linears with
residual epilogue, RMSNorm backward with the residual gradient."""
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
    # `python tools/sanitize.py kernels`: the kernel-level calls only (racecheck
    # is too slow for the threaded pipeline run, whose emit timeout then fires)
    if sys.argv[1:2] != ["kernels"]:
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
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    T, h, N = 300, 64, 264  # ragged: partial row and column tiles
    xm = torch.randn(T, h, device="cuda").bfloat16()
    w1 = (torch.randn(h, N, device="cuda") * 0.1).bfloat16()
    w2 = (torch.randn(N, h, device="cuda") * 0.1).bfloat16()
    pre = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    act, dpre = torch.empty_like(pre), torch.empty_like(pre)
    call("ee_mlp_up_gelu", ptr(xm), ptr(w1), T, h, N, ptr(pre), ptr(act), stream_ptr())
    call("ee_mlp_gelu_bwd", ptr(xm), ptr(w2), T, h, N, ptr(pre), ptr(dpre), stream_ptr())
    acc = torch.zeros(h, N, device="cuda")
    call("ee_wgrad_accum", ptr(xm), ptr(dpre), T, h, N, ptr(acc), stream_ptr())
    nh, dh, smax = 4, 128, 2048  # rows spanning several chunks -> k_attn_rows128
    kc = torch.randn(smax, nh * dh, device="cuda").bfloat16()
    vc = torch.randn(smax, nh * dh, device="cuda").bfloat16()
    q = torch.randn(5, nh * dh, device="cuda")
    pos = torch.tensor([700, 1023, 1500, 2000, 2047], dtype=torch.int32, device="cuda")
    out = torch.empty(5, nh * dh, dtype=torch.bfloat16, device="cuda")
    wsb = _lib.load().ee_workspace_bytes(_lib.EE_OP_ATTENTION, 5, nh * dh, 0, nh, smax)
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    call("ee_decode_attention", ptr(q), 5, ptr(pos), 2047, ptr(kc), ptr(vc), nh, dh,
         _lib.EE_BF16, ptr(out), ptr(ws), wsb, stream_ptr())
    # training attention (tcgen05, TMEM-operand backward), small shape
    Bt, St, Ht = 1, 256, 1
    ht = Ht * 128
    qa, ka, va, doa = (torch.randn(Bt * St, ht, device="cuda").bfloat16() for _ in range(4))
    oa = torch.empty_like(qa)
    lse = torch.empty(Bt, Ht, St, device="cuda")
    call("ee_attn_train_fwd", ptr(qa), ht, ptr(ka), ht, ptr(va), ht, Bt, St, Ht, ptr(oa), ht,
         ptr(lse), stream_ptr())
    dqa, dka, dva = torch.empty_like(qa), torch.empty_like(qa), torch.empty_like(qa)
    dsum = torch.empty_like(lse)
    call("ee_attn_train_bwd", ptr(qa), ht, ptr(ka), ht, ptr(va), ht, ptr(oa), ht, ptr(doa), ht,
         ptr(lse), Bt, St, Ht, ptr(dqa), ht, ptr(dka), ht, ptr(dva), ht, ptr(dsum), stream_ptr())
    # backbone linears with the residual epilogue (ragged tiles)
    yl = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    call("ee_linear_fwd", ptr(xm), ptr(w1), T, h, N, ptr(pre), ptr(yl), stream_ptr())
    gl = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    call("ee_linear_dgrad", ptr(dpre), ptr(w1), T, h, N, ptr(xm), ptr(gl), stream_ptr())
    # RMSNorm backward joining the residual branch's gradient
    from paper_2312_04916_b200.training import rmsnorm_fork
    xf = torch.randn(37, 264, device="cuda").bfloat16().requires_grad_()
    wf = torch.ones(264, device="cuda", requires_grad=True)
    yf, xa = rmsnorm_fork(xf, wf)
    torch.autograd.backward([yf, xa], [torch.ones_like(yf), torch.ones_like(xa)])
    p = {"a": torch.zeros(1003, device="cuda")}
    Adam(1e-3).step(p, {"a": torch.ones(1003, device="cuda")}, 0.5)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
