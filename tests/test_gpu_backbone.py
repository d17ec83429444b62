"""Training-backbone kernels against the float64 oracle: the fused RMSNorm
forward/backward (`ee_rmsnorm_fwd/bwd`, csrc/rmsnorm_train.cu), the
reference's `rmsnorm_fwd` / `rmsnorm_bwd` boundary kernels
(eepipe/_pykernels.py:36-49).

Tolerances: bf16 outputs (y, gx) within 1e-2 relative (Frobenius; one bf16
rounding), float32 statistics inv_rms within 1e-5 and the float32 weight
gradient within 1e-4 relative; the oracle runs on the bf16-rounded inputs.
The weight gradient is deterministic (fixed-order reduction): bitwise equal
across calls.
"""
import numpy as np
import pytest

import ee_oracle as O

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("n,h", [(1, 8), (37, 264), (4096, 2048), (1000, 5120), (16, 7168)])
def test_rmsnorm_fwd_bwd_match_oracle(n, h):
    import torch
    from paper_2312_04916_b200.training import rmsnorm
    rng = np.random.default_rng(n * 7 + h)
    x = torch.tensor(rng.normal(size=(n, h)) * 3.0, dtype=torch.bfloat16, device="cuda")
    w = torch.tensor(rng.normal(1.0, 0.2, size=h), dtype=torch.float32, device="cuda")
    g = torch.tensor(rng.normal(size=(n, h)), dtype=torch.bfloat16, device="cuda")
    xr = x.clone().requires_grad_()
    wr = w.clone().requires_grad_()
    y = rmsnorm(xr, wr)
    y.backward(g)
    x64, w64, g64 = (t.double().cpu().numpy() for t in (x, w, g))
    ry, rinv = O.rmsnorm_fwd(x64, w64)
    rgx, rgw = O.rmsnorm_bwd(x64, w64, rinv, g64)
    assert y.dtype == torch.bfloat16
    assert _rel(y.double().detach().cpu().numpy(), ry) < 1e-2
    assert _rel(xr.grad.double().cpu().numpy(), rgx) < 1e-2
    assert _rel(wr.grad.double().cpu().numpy(), rgw) < 1e-4
    # determinism of the fixed-order weight-gradient reduction
    wr2 = w.clone().requires_grad_()
    rmsnorm(x.clone().requires_grad_(), wr2).backward(g)
    assert torch.equal(wr.grad, wr2.grad)


def test_rmsnorm_inv_rms_statistics():
    import ctypes
    import torch
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    rng = np.random.default_rng(0)
    n, h = 64, 4096
    x = torch.tensor(rng.normal(size=(n, h)), dtype=torch.bfloat16, device="cuda")
    w = torch.ones(h, device="cuda")
    y = torch.empty_like(x)
    inv = torch.empty(n, device="cuda")
    call("ee_rmsnorm_fwd", ptr(x), n, h, ptr(w), ctypes.c_float(1e-6), ptr(y), ptr(inv),
         stream_ptr())
    _, rinv = O.rmsnorm_fwd(x.double().cpu().numpy(), np.ones(h))
    assert np.abs(inv.cpu().numpy() - rinv).max() / rinv.max() < 1e-5


@pytest.mark.parametrize("T,K,N", [(5, 32, 32), (4096, 2048, 2048), (4096, 8192, 2048),
                                   (2048, 5120, 15360), (300, 264, 776)])
def test_linear_fwd_dgrad_match_fp32(T, K, N):
    """Backbone linears on the tcgen05 GEMM (ee_linear_fwd / ee_linear_dgrad,
    csrc/linear_train.cu) against a float32 torch reference on the same bf16
    inputs: Y = X W + R and dX = dY W^T within 1e-2 relative (Frobenius; one
    bf16 rounding of a float32 accumulation), the residual added before the
    rounding."""
    import torch
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    g = torch.Generator(device="cuda").manual_seed(T + K + N)
    x = torch.randn(T, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(K, N, device="cuda", generator=g) * 0.02).bfloat16()
    r = torch.randn(T, N, device="cuda", generator=g).bfloat16()
    gy = torch.randn(T, N, device="cuda", generator=g).bfloat16()
    y = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    gx = torch.empty(T, K, device="cuda", dtype=torch.bfloat16)
    _lib.load()
    call("ee_linear_fwd", ptr(x), ptr(w), T, K, N, ptr(r), ptr(y), stream_ptr())
    call("ee_linear_dgrad", ptr(gy), ptr(w), T, K, N, None, ptr(gx), stream_ptr())
    torch.cuda.synchronize()
    ry = x.float() @ w.float() + r.float()
    rgx = gy.float() @ w.float().t()
    assert _rel(y.double().cpu().numpy(), ry.double().cpu().numpy()) < 1e-2
    assert _rel(gx.double().cpu().numpy(), rgx.double().cpu().numpy()) < 1e-2
    y0 = torch.empty_like(y)
    call("ee_linear_fwd", ptr(x), ptr(w), T, K, N, None, ptr(y0), stream_ptr())
    torch.cuda.synchronize()
    assert _rel(y0.double().cpu().numpy(), (x.float() @ w.float()).double().cpu().numpy()) < 1e-2


@pytest.mark.parametrize("kind,T,K,N", [("fwd", 8192, 4096, 1024), ("fwd", 8000, 4096, 1000),
                                        ("wgrad", 4096, 4096, 1280), ("wgrad", 4000, 4096, 1272)])
def test_gemm_stream_k_tail_matches_fp32_and_repeats(kind, T, K, N):
    """The CTA-pair GEMM's stream-K tail (tc_gemm.cuh: the last wave's tiles'
    k-blocks spread over all clusters, owners adding lower clusters' fp32
    partials) on shapes that take it (a partial last wave, >= 64 k-blocks),
    two with ragged edges: Y = X W (ee_linear_fwd, 128 tiles x 64 k-blocks)
    against float32 torch within 1e-2, and dW += X^T dY (ee_wgrad_accum,
    80 tiles, float32 TMA reduce-add in place) within 1e-3 of the float64
    reference; a second run is bitwise equal (fixed summation order)."""
    import torch
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    _lib.load()
    g = torch.Generator(device="cuda").manual_seed(7 * T + K + N)
    x = torch.randn(T, K, device="cuda", generator=g).bfloat16()
    if kind == "fwd":
        w = (torch.randn(K, N, device="cuda", generator=g) * 0.02).bfloat16()
        y1 = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
        y2 = torch.empty_like(y1)
        call("ee_linear_fwd", ptr(x), ptr(w), T, K, N, None, ptr(y1), stream_ptr())
        call("ee_linear_fwd", ptr(x), ptr(w), T, K, N, None, ptr(y2), stream_ptr())
        torch.cuda.synchronize()
        ref = x.float() @ w.float()
        assert _rel(y1.double().cpu().numpy(), ref.double().cpu().numpy()) < 1e-2
        assert torch.equal(y1, y2)
    else:
        dy = torch.randn(T, N, device="cuda", generator=g).bfloat16()
        dw0 = torch.randn(K, N, device="cuda", generator=g)
        dw1, dw2 = dw0.clone(), dw0.clone()
        call("ee_wgrad_accum", ptr(x), ptr(dy), T, K, N, ptr(dw1), stream_ptr())
        call("ee_wgrad_accum", ptr(x), ptr(dy), T, K, N, ptr(dw2), stream_ptr())
        torch.cuda.synchronize()
        rdw = dw0.double() + x.double().t() @ dy.double()
        assert _rel(dw1.double().cpu().numpy(), rdw.cpu().numpy()) < 1e-3
        assert torch.equal(dw1, dw2)


@pytest.mark.parametrize("T,K,N,P", [(300, 256, 256, 3), (4096, 2048, 2048, 3),
                                     (2000, 5120, 5120, 3), (8192, 2048, 2048, 2)])
def test_stacked_linears_match_fp32(T, K, N, P):
    """q / k / v as ONE GEMM each way over P adjacent (K, N) weight matrices
    (ee_linear_fwd_stacked / ee_linear_dgrad_stacked / ee_wgrad_accum_stacked,
    tc_gemm.cuh stacked operands): Y = X [W_0 | ...] and dX = dY [W_0 | ...]^T
    within 1e-2 of float32 torch (one bf16 rounding), dW_j += X^T dY_j in
    float32 within 1e-3 of float64 into P adjacent accumulators; the memory
    around each block is untouched."""
    import torch
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    _lib.load()
    g = torch.Generator(device="cuda").manual_seed(T + K + N + P)
    x = torch.randn(T, K, device="cuda", generator=g).bfloat16()
    w = (torch.randn(P, K, N, device="cuda", generator=g) * 0.02).bfloat16()
    wcat = torch.cat(list(w), dim=1).float()                      # (K, P N)
    y = torch.empty(T, P * N, device="cuda", dtype=torch.bfloat16)
    call("ee_linear_fwd_stacked", ptr(x), ptr(w), T, K, N, P, ptr(y), stream_ptr())
    gy = torch.randn(T, P * N, device="cuda", generator=g).bfloat16()
    r = torch.randn(T, K, device="cuda", generator=g).bfloat16()
    gx = torch.empty(T, K, device="cuda", dtype=torch.bfloat16)
    call("ee_linear_dgrad_stacked", ptr(gy), ptr(w), T, K, N, P, ptr(r), ptr(gx), stream_ptr())
    guard = 4096
    acc = torch.randn(P * K * N + 2 * guard, device="cuda", generator=g)
    acc0 = acc.clone()
    call("ee_wgrad_accum_stacked", ptr(x), ptr(gy), T, K, N, P, ptr(acc[guard:]), stream_ptr())
    torch.cuda.synchronize()
    ry = x.float() @ wcat
    rgx = gy.float() @ wcat.t() + r.float()
    assert _rel(y.double().cpu().numpy(), ry.double().cpu().numpy()) < 1e-2
    assert _rel(gx.double().cpu().numpy(), rgx.double().cpu().numpy()) < 1e-2
    dw = acc[guard:guard + P * K * N].view(P, K, N).double()
    for j in range(P):
        ref = acc0[guard + j * K * N:guard + (j + 1) * K * N].view(K, N).double() + \
            x.double().t() @ gy[:, j * N:(j + 1) * N].double()
        assert _rel(dw[j].cpu().numpy(), ref.cpu().numpy()) < 1e-3, j
    assert torch.equal(acc[:guard], acc0[:guard]) and torch.equal(acc[-guard:], acc0[-guard:])


def test_stacked_qkv_training_path_matches_separate():
    """The training block with q / k / v fused (one stacked GEMM each way, q /
    k / v and their gradients as column blocks of one buffer read in place by
    the attention kernels) against the three-GEMM path (EE_STACKED_QKV=0
    semantics): loss and every float32 gradient sum within bf16 tolerance
    (2e-2 relative per tensor)."""
    import torch
    from paper_2312_04916_b200 import training as TR
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model
    cfg = ModelConfig(2, 512, 4, 1024, 256, exits=(ExitSpec(1, "minimalistic", 0.5),))
    model = build_model(cfg, 0)
    tokens = np.random.default_rng(3).integers(0, 1024, size=(2, 257))
    out = {}
    for stacked in (True, False):
        TR._STACKED_QKV = stacked
        uses0 = TR._STACKED_USES[0]
        try:
            tm = TR.TrainModel(model, master_dtype=torch.float32)
            tm.zero_grad()
            total, per_exit = TR.weighted_loss(tm, tokens, [1.0] * len(tm.heads))
            total.backward()
            TR.join_wgrad()
            assert TR._STACKED_USES[0] - uses0 == (cfg.num_layers if stacked else 0)
            torch.cuda.synchronize()
            out[stacked] = (dict(enumerate(per_exit)),
                            {k: v.detach().cpu().clone() for k, v in tm.main_grads.items()})
        finally:
            TR._STACKED_QKV = True
    (la, ga), (lb, gb) = out[True], out[False]
    for k in lb:
        assert abs(la[k] - lb[k]) <= 1e-2 * abs(lb[k]), k
    for k in gb:
        if "wq" in k or "wk" in k or "wv" in k or "wo" in k or "w1" in k:
            assert _rel(ga[k].numpy().astype(np.float64), gb[k].numpy().astype(np.float64)) < 2e-2, k


@pytest.mark.parametrize("n,h", [(37, 264), (4096, 2048), (1000, 5120)])
def test_rmsnorm_fork_joins_residual_gradient(n, h):
    """`rmsnorm_fork` (ee_rmsnorm_bwd with gres): the residual branch's
    gradient of x is added inside the RMSNorm backward kernel.  x.grad must
    equal the float64 oracle's rmsnorm_bwd + the residual gradient (1e-2,
    bf16 output), and the weight gradient must not change (1e-4)."""
    import torch
    from paper_2312_04916_b200.training import rmsnorm_fork
    rng = np.random.default_rng(n + h)
    x = torch.tensor(rng.normal(size=(n, h)) * 2.0, dtype=torch.bfloat16, device="cuda")
    w = torch.tensor(rng.normal(1.0, 0.2, size=h), dtype=torch.float32, device="cuda")
    g = torch.tensor(rng.normal(size=(n, h)), dtype=torch.bfloat16, device="cuda")
    gr = torch.tensor(rng.normal(size=(n, h)), dtype=torch.bfloat16, device="cuda")
    xr = x.clone().requires_grad_()
    wr = w.clone().requires_grad_()
    y, xa = rmsnorm_fork(xr, wr)
    torch.autograd.backward([y, xa], [g, gr])
    x64, w64, g64 = (t.double().cpu().numpy() for t in (x, w, g))
    _, rinv = O.rmsnorm_fwd(x64, w64)
    rgx, rgw = O.rmsnorm_bwd(x64, w64, rinv, g64)
    rgx = rgx + gr.double().cpu().numpy()
    assert _rel(xr.grad.double().cpu().numpy(), rgx) < 1e-2
    assert _rel(wr.grad.double().cpu().numpy(), rgw) < 1e-4
