"""GPU training path: weighted multi-exit loss with fused tcgen05 heads, the
single-device gradient oracle and the threaded 1F1B pipeline executor.

Reference anchors: `single_device_gradients` golden (tests/golden wl_*,
produced by the reference's float64 autodiff) — compared at bf16 tolerance
(per-exit losses within 2e-2 relative, gradients within 1e-1 relative in
Frobenius norm: the whole backbone runs in bf16); pipeline vs single-device
on the GPU — same kernels, so they must agree to 1e-3 relative (the
reference's own check is < 1e-9 in float64, tests/test_pipeline.py:59-69).
"""
import numpy as np
import pytest

from helpers import arrays, gold
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

pytestmark = pytest.mark.gpu


def _wl_model():
    cfg = ModelConfig(4, 32, 4, 64, 16, exits=(ExitSpec(1, loss_weight=0.25),
                                               ExitSpec(2, "norm+embed", 0.5)),
                      tie_embeddings=True)
    return build_model(cfg, 3)


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_weighted_loss_gradients_match_reference():
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    m = _wl_model()
    tm = TrainModel(m)
    batch = arrays()["wl_batch"]
    grads, per_exit = single_device_gradients(tm, batch, [0.25, 0.5, 1.0], 2)
    ref_loss = gold()["wl_per_exit"]
    for k, v in ref_loss.items():
        assert per_exit[k] == pytest.approx(v, rel=2e-2), k
    a = arrays()
    for name, g in grads.items():
        ref = a[f"wl_grad::{name}"]
        assert _rel(g.float().cpu().numpy(), ref) < 1e-1, name


def test_pipeline_matches_single_device():
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    cfg = ModelConfig(8, 64, 4, 128, 16, exits=(ExitSpec(2, loss_weight=0.3),
                                                ExitSpec(4, "norm+embed", 0.6)))
    m = build_model(cfg, 1)
    batch = np.random.default_rng(2).integers(0, 128, size=(8, 17))
    ref, ref_loss = single_device_gradients(TrainModel(m), batch, [0.3, 0.6, 1.0], 2)
    for P in (2, 4):
        grads, rep = run_iteration_1f1b(partition(m, P), batch, IterationOptions(2), model=m)
        assert set(grads) == set(ref)
        for n in ref:
            assert _rel(grads[n].float().cpu().numpy(), ref[n].float().cpu().numpy()) < 1e-3, n
        for k, v in ref_loss.items():
            assert rep.per_exit_losses[k] == pytest.approx(v, rel=1e-3)
        for s in range(1, P + 1):
            assert rep.max_in_flight[s] == min(P - s + 1, 4)
        assert all(rep.activation_messages[s] == 4 for s in range(1, P))
        assert all(rep.gradient_messages[s] == 4 for s in range(2, P + 1))


def test_tied_pipeline_sums_replicas():
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    m = _wl_model()
    batch = arrays()["wl_batch"]
    ref, _ = single_device_gradients(TrainModel(m), batch, [0.25, 0.5, 1.0], 2)
    part = partition(m, 2)
    assert "tok_emb" in part.tied_replicas
    grads, _ = run_iteration_1f1b(part, batch, IterationOptions(2), model=m)
    # the replicas' bf16 gradients are summed after the iteration instead of
    # accumulating inside one autograd graph: bf16 rounding order differs
    assert _rel(grads["tok_emb"].float().cpu().numpy(), ref["tok_emb"].float().cpu().numpy()) < 1e-2
    for n in ref:
        if n != "tok_emb":
            assert _rel(grads[n].float().cpu().numpy(), ref[n].float().cpu().numpy()) < 1e-3, n


def test_mixed_precision_fused_wgrad_matches_plain():
    """Mixed mode (float32 gradient sums; the backbone's linear layers add
    their weight gradients straight into them with `ee_wgrad_accum`) against
    the plain bf16 model: same gradients within bf16 tolerance (2e-2), for the
    single-device oracle and the 2-stage pipeline."""
    import torch
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import TrainModel, single_device_gradients
    cfg = ModelConfig(4, 64, 4, 128, 16, exits=(ExitSpec(1, loss_weight=0.3),
                                                ExitSpec(2, "norm+embed", 0.6)))
    m = build_model(cfg, 5)
    batch = np.random.default_rng(6).integers(0, 128, size=(8, 17))
    ref, _ = single_device_gradients(TrainModel(m), batch, [0.3, 0.6, 1.0], 2)
    mixed, _ = single_device_gradients(TrainModel(m, master_dtype=torch.float32), batch,
                                       [0.3, 0.6, 1.0], 2)
    grads, _ = run_iteration_1f1b(partition(m, 2), batch, IterationOptions(2), model=m,
                                  master_dtype=torch.float32)
    for n in ref:
        r = ref[n].float().cpu().numpy()
        assert _rel(mixed[n].cpu().numpy(), r) < 2e-2, n
        assert _rel(grads[n].cpu().numpy(), r) < 2e-2, n
    # the fused path really ran: layer weights carry no bf16 .grad
    tm = TrainModel(m, master_dtype=torch.float32)
    single_device_gradients(tm, batch, [0.3, 0.6, 1.0], 2)
    assert tm.params["layer1.w1"].grad is None
    assert float(tm.main_grads["layer1.w1"].abs().sum()) > 0


@pytest.mark.parametrize("T,h,N", [(300, 64, 264), (4096, 2048, 8192)])
def test_mlp_gelu_fused_gemms_match_torch(T, h, N):
    """ee_mlp_up_gelu / ee_mlp_gelu_bwd (GELU fused into tcgen05 GEMM
    epilogues, csrc/mlp_train.cu) against a float32 torch restatement on the
    same bf16 inputs: pre, act and dpre within 1e-2 relative (Frobenius; bf16
    outputs), ragged T / N included."""
    import torch
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    g = torch.Generator(device="cuda").manual_seed(T + N)
    x = (torch.randn(T, h, device="cuda", generator=g)).bfloat16()
    w1 = (torch.randn(h, N, device="cuda", generator=g) * h ** -0.5).bfloat16()
    w2 = (torch.randn(N, h, device="cuda", generator=g) * N ** -0.5).bfloat16()
    dy = torch.randn(T, h, device="cuda", generator=g).bfloat16()
    pre = torch.empty(T, N, dtype=torch.bfloat16, device="cuda")
    act = torch.empty_like(pre)
    dpre = torch.empty_like(pre)
    call("ee_mlp_up_gelu", ptr(x), ptr(w1), T, h, N, ptr(pre), ptr(act), stream_ptr())
    call("ee_mlp_gelu_bwd", ptr(dy), ptr(w2), T, h, N, ptr(pre), ptr(dpre), stream_ptr())
    torch.cuda.synchronize()
    ref_pre = x.float() @ w1.float()
    ref_act = torch.nn.functional.gelu(ref_pre)
    p = ref_pre.clone().requires_grad_()
    torch.nn.functional.gelu(p).backward(dy.float() @ w2.float().t())
    rel = lambda a, b: float((a.float() - b).norm() / b.norm())  # noqa: E731
    assert rel(pre, ref_pre) < 1e-2
    assert rel(act, ref_act) < 1e-2
    assert rel(dpre, p.grad) < 1e-2


def test_mixed_precision_own_kernels_match_fp32_reference():
    """The mixed-precision training path that the C2 bench times (bf16 leaves,
    float32 gradient sums; every backbone linear, the causal attention
    (head_dim 128, S = 128), the fused RMSNorm / residual-gradient kernels and
    the fused exit heads are own sm_100a kernels) against a float32 torch
    autograd reference of the SAME bf16-rounded weights.  Per-tensor
    tolerance 3e-2 relative (Frobenius): bf16 activations between kernels,
    float32 accumulation -- tight enough that a wrong scale factor on any
    tensor (>= 2x) fails.  Per-exit losses within 1e-2."""
    import torch
    import torch.nn.functional as F
    from paper_2312_04916_b200.training import NORM_EPS, TrainModel, single_device_gradients
    cfg = ModelConfig(2, 256, 2, 512, 256, exits=(ExitSpec(1, "minimalistic", 0.3),))
    m = build_model(cfg, 5)
    batch = np.random.default_rng(7).integers(0, 512, size=(2, 129))
    weights = [0.3, 1.0]
    tm = TrainModel(m, master_dtype=torch.float32)
    grads, per_exit = single_device_gradients(tm, batch, weights, 2)

    P = {n: p.detach().float().clone().requires_grad_() for n, p in tm.params.items()}

    def rms(x, w):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + NORM_EPS) * w

    tok = torch.as_tensor(batch, device="cuda")
    inp, tgt = tok[:, :-1], tok[:, 1:]
    B, S = inp.shape
    x = P["tok_emb"][inp] + P["pos_emb"][torch.arange(S, device="cuda")][None]
    taps = {}
    for i in range(1, cfg.num_layers + 1):
        pre = f"layer{i}"
        h1 = rms(x, P[f"{pre}.attn_norm"])
        split = lambda t: t.view(B, S, cfg.num_heads, -1).transpose(1, 2)  # noqa: E731
        q, k, v = (split(h1 @ P[f"{pre}.{w}"]) for w in ("wq", "wk", "wv"))
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + a.transpose(1, 2).reshape(B, S, -1) @ P[f"{pre}.wo"]
        h2 = rms(x, P[f"{pre}.mlp_norm"])
        x = x + F.gelu(h2 @ P[f"{pre}.w1"]) @ P[f"{pre}.w2"]
        taps[i] = x
    total, ref_exit = 0.0, {}
    for hd, w in zip(tm.heads, weights):
        xi = taps[hd.layer_index]
        if "norm" in hd.param_names:
            xi = rms(xi, P[hd.param_names["norm"]])
        logits = xi @ P[hd.param_names["out"]].t()
        ce = F.cross_entropy(logits.reshape(-1, logits.shape[-1]), tgt.reshape(-1))
        ref_exit[hd.key] = float(ce.detach())
        total = total + w * ce
    total.backward()
    for key, v in ref_exit.items():
        assert per_exit[key] == pytest.approx(v, rel=1e-2), key
    for name, g in grads.items():
        assert _rel(g.float().cpu().numpy(), P[name].grad.double().cpu().numpy()) < 3e-2, name
