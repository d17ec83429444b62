"""Training-backbone causal attention on tcgen05 (ee_attn_train_fwd / _bwd,
csrc/attention_train.cu) against a float32 torch reference of the same
causal softmax attention on the same bf16 inputs (eepipe/autodiff.py:265-298;
the reference's attention_fwd / attention_bwd, eepipe/_pykernels.py:52-62):
output within 1e-2 relative (Frobenius: bf16 P and one bf16 rounding of
the output), gradients within 2e-2 (bf16 P and dS operands), lse within
1e-4 absolute; a second call is bitwise identical (no atomics).  Shapes cover
one tile, several tiles and batches, the C2 layer (B 2, S 2048, 16 heads) and
the C4 layer (40 heads), and inputs read in place from a fused (T, 3h)
projection buffer (row stride 3h)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def _ref(q, k, v, B, S, H):
    """float32 causal attention on (B*S, H*128) row-major q/k/v views."""
    import torch
    qf, kf, vf = (t.float().reshape(B, S, H, 128).transpose(1, 2) for t in (q, k, v))
    s = (qf @ kf.transpose(-1, -2)) / np.sqrt(128.0)
    mask = torch.ones(S, S, dtype=torch.bool, device=q.device).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    p = torch.softmax(s, -1)
    o = p @ vf
    return o.transpose(1, 2).reshape(B * S, H * 128), lse


@pytest.mark.parametrize("B,S,H,fused", [(1, 128, 1, False), (2, 384, 2, False),
                                         (2, 2048, 16, False), (1, 2048, 40, False),
                                         (2, 512, 4, True)])
def test_attention_train_fwd_bwd_match_fp32(B, S, H, fused):
    import torch
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200._lib import call, ptr, stream_ptr
    _lib.load()
    h = H * 128
    T = B * S
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + S + H)
    if fused:
        qkv = torch.randn(T, 3 * h, device="cuda", generator=g).bfloat16()
        q, k, v = qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:]
        ld = 3 * h
    else:
        q, k, v = (torch.randn(T, h, device="cuda", generator=g).bfloat16() for _ in range(3))
        ld = h
    do = torch.randn(T, h, device="cuda", generator=g).bfloat16()
    o = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device="cuda", dtype=torch.float32)
    call("ee_attn_train_fwd", ptr(q), ld, ptr(k), ld, ptr(v), ld, B, S, H, ptr(o), h, ptr(lse),
         stream_ptr())
    dq, dk, dv = (torch.empty(T, h, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    dsum = torch.empty(B, H, S, device="cuda", dtype=torch.float32)
    call("ee_attn_train_bwd", ptr(q), ld, ptr(k), ld, ptr(v), ld, ptr(o), h, ptr(do), h, ptr(lse),
         B, S, H, ptr(dq), h, ptr(dk), h, ptr(dv), h, ptr(dsum), stream_ptr())
    torch.cuda.synchronize()
    qr, kr, vr = (t.detach().float().clone().requires_grad_() for t in (q, k, v))
    ro, rlse = _ref(qr, kr, vr, B, S, H)
    ro.backward(do.float())
    assert _rel(o, ro.detach()) < 1e-2
    assert (lse - rlse.detach()).abs().max().item() < 1e-4 * max(1.0, rlse.abs().max().item())
    assert _rel(dv, vr.grad) < 2e-2
    assert _rel(dk, kr.grad) < 2e-2
    assert _rel(dq, qr.grad) < 2e-2
    # deterministic: a second call gives the same bits
    o2, dq2 = torch.empty_like(o), torch.empty_like(dq)
    call("ee_attn_train_fwd", ptr(q), ld, ptr(k), ld, ptr(v), ld, B, S, H, ptr(o2), h, ptr(lse),
         stream_ptr())
    call("ee_attn_train_bwd", ptr(q), ld, ptr(k), ld, ptr(v), ld, ptr(o2), h, ptr(do), h, ptr(lse),
         B, S, H, ptr(dq2), h, ptr(dk), h, ptr(dv), h, ptr(dsum), stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(dq, dq2)
