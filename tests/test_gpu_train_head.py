"""GPU parity of the fused tcgen05 training exit head against the float64
oracle (oracle/ee_oracle.py:exit_head_train, itself pinned to the reference's
autodiff in tests/test_oracle_golden.py).

Tolerances (bf16 inputs, fp32 accumulation, bf16 logit gradient): loss within
1e-3 relative (north star); gradients within 2e-2 relative in Frobenius norm
(the logit gradient is rounded to bf16 before the two backward GEMMs).
The oracle runs on the bf16-rounded inputs, so the tolerance measures the
kernel, not the input cast.
"""
import numpy as np
import pytest

import ee_oracle as O
from helpers import arrays

pytestmark = pytest.mark.gpu


def _run(x, w, t, weight=1.0):
    import torch
    from paper_2312_04916_b200.training import exit_head_loss_and_grads
    xd = torch.from_numpy(x).cuda().bfloat16()
    wd = torch.from_numpy(w).cuda().bfloat16()
    td = torch.from_numpy(np.asarray(t, dtype=np.int64)).cuda()
    loss, dx, dw = exit_head_loss_and_grads(xd, wd, td, weight)
    torch.cuda.synchronize()
    xr = xd.float().cpu().numpy().astype(np.float64)
    wr = wd.float().cpu().numpy().astype(np.float64)
    return float(loss), dx.cpu().numpy(), dw.cpu().numpy(), xr, wr


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_train_head_golden_small():
    a = arrays()
    x, w, t = a["ce_x"], a["ce_w"], a["ce_targets"]
    loss, dx, dw, xr, wr = _run(x, w, t)
    rl, rdx, rdw, _ = O.exit_head_train(xr, wr, t)
    assert loss == pytest.approx(rl, rel=1e-3)
    assert _rel(dx, rdx) < 2e-2
    assert _rel(dw, rdw) < 2e-2
    # the reference's own (float64) loss on the unrounded inputs, looser
    assert loss == pytest.approx(float(a["ce_min_loss"]), rel=2e-2)


@pytest.mark.parametrize("n,h,V,weight", [(256, 512, 1000, 1.0), (384, 256, 4096, 0.25),
                                          (136, 1024, 2056, 0.5), (12, 16, 32, 1.0),
                                          (301, 64, 520, 0.7)])
def test_train_head_random(n, h, V, weight):
    rng = np.random.default_rng(n + V)
    x = rng.normal(size=(n, h)).astype(np.float32)
    w = (rng.normal(size=(V, h)) * 0.05).astype(np.float32)
    t = rng.integers(0, V, size=n)
    loss, dx, dw, xr, wr = _run(x, w, t, weight)
    rl, rdx, rdw, _ = O.exit_head_train(xr, wr, t, weight)
    assert loss == pytest.approx(rl, rel=1e-3)
    assert _rel(dx, rdx) < 2e-2
    assert _rel(dw, rdw) < 2e-2


def test_train_head_deterministic_and_accumulates():
    import torch
    from paper_2312_04916_b200.training import exit_head_loss_and_grads
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.normal(size=(128, 256)).astype(np.float32)).cuda().bfloat16()
    w = torch.from_numpy((rng.normal(size=(512, 256)) * 0.05).astype(np.float32)).cuda().bfloat16()
    t = torch.from_numpy(rng.integers(0, 512, size=128)).cuda()
    l1, dx1, dw1 = exit_head_loss_and_grads(x, w, t)
    l2, dx2, dw2 = exit_head_loss_and_grads(x, w, t)
    assert float(l1) == float(l2)
    assert torch.equal(dx1, dx2) and torch.equal(dw1, dw2)
    acc = torch.zeros_like(dw1)
    exit_head_loss_and_grads(x, w, t, dw_acc=acc)
    exit_head_loss_and_grads(x, w, t, dw_acc=acc)
    assert torch.allclose(acc, 2 * dw1, rtol=1e-6, atol=1e-12)


def test_train_head_rejects_bad_targets():
    import torch
    from paper_2312_04916_b200.errors import TokenError
    from paper_2312_04916_b200.training import exit_head_loss_and_grads
    x = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(16, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(TokenError):
        exit_head_loss_and_grads(x, w, torch.full((8,), 16, dtype=torch.int64, device="cuda"))


def test_train_head_ordered_split_k_matches_oracle_and_is_deterministic():
    """A long vocabulary (V = 16384: 256 k-blocks) with few dX tiles makes the
    dX GEMM use the ordered split-K path (per-region acquire/release flags,
    exit_head_train.cu): same tolerance as above, and bitwise reproducible."""
    import torch
    from paper_2312_04916_b200.training import exit_head_loss_and_grads
    rng = np.random.default_rng(11)
    n, h, V = 512, 256, 16384
    x = rng.normal(size=(n, h)).astype(np.float32)
    w = (rng.normal(size=(V, h)) * 0.05).astype(np.float32)
    t = rng.integers(0, V, size=n)
    loss, dx, dw, xr, wr = _run(x, w, t, 0.5)
    rl, rdx, rdw, _ = O.exit_head_train(xr, wr, t, 0.5)
    assert loss == pytest.approx(rl, rel=1e-3)
    assert _rel(dx, rdx) < 2e-2
    assert _rel(dw, rdw) < 2e-2
    _, dx2, _, _, _ = _run(x, w, t, 0.5)
    assert np.array_equal(dx, dx2)


def test_split_forward_backward_matches_fused():
    """ee_exit_head_train_fwd / _bwd (the head split at the autograd
    boundary, used in mixed precision): the forward's loss equals the fused
    call's bitwise; the backward with an incoming gradient g read from device
    memory gives g * dx and adds g * dW into an existing float32 sum."""
    import torch
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    from paper_2312_04916_b200.training import exit_head_loss_and_grads
    g = torch.Generator(device="cuda").manual_seed(3)
    n, h, V = 300, 256, 1000
    x = torch.randn(n, h, device="cuda", generator=g).bfloat16()
    W = (torch.randn(V, h, device="cuda", generator=g) * 0.05).bfloat16()
    t = torch.randint(0, V, (n,), device="cuda", generator=g)
    loss, dx, dw = exit_head_loss_and_grads(x, W, t.cpu().numpy(), 0.6)
    lib = _lib.load()
    wsb = lib.ee_workspace_bytes(_lib.EE_OP_EXIT_HEAD_TRAIN, n, h, V, 0, 0)
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    G = torch.empty(n, V, dtype=torch.bfloat16, device="cuda")
    loss2 = torch.zeros((), device="cuda")
    call("ee_exit_head_train_fwd", ptr(x), n, h, ptr(W), V, ptr(t), 0.6, ptr(loss2), ptr(G),
         ptr(ws), wsb, stream_ptr())
    gs = torch.tensor(0.7, device="cuda")
    dx2 = torch.empty(n, h, device="cuda")
    acc = torch.ones(V, h, device="cuda")
    call("ee_exit_head_train_bwd", ptr(x), n, h, ptr(W), V, ptr(G), ptr(gs), ptr(dx2), ptr(acc),
         ptr(ws), wsb, stream_ptr())
    torch.cuda.synchronize()
    assert float(loss2) == float(loss)
    assert torch.allclose(dx2, 0.7 * dx, rtol=1e-5, atol=1e-7)
    assert torch.allclose(acc - 1.0, 0.7 * dw, rtol=1e-4, atol=1e-6)
