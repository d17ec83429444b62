"""Fused multi-tensor optimizer (`ee_optimizer_step`, csrc/optim.cu) and the
training loop (`training.train`) against the reference.

* Kernel parity: SGD / Adam over tensors of ragged sizes, float32 and bf16
  gradients, several steps, against the float64 restatement of
  `SGD.step` / `Adam.step` (oracle.sgd_step / adam_step, eepipe/training.py:
  24-53) fed the same gradients: parameters within 1e-5 relative (float32
  arithmetic of the same update).
* Loop parity: `train` for 3 Adam steps from the reference's initialisation
  on the reference's own batches (tests/golden/trained.npz) against the
  reference's `train` (tests/golden/trained.json): per-exit losses of every
  step within 2e-2 relative and parameters after 3 steps within 10% of the
  reference's Adam displacement (bf16 compute, float32 gradients, the
  reference is float64; Adam's normalised step turns the bf16-level noise of
  near-zero gradients — rare embedding rows — into full-size steps, so the
  bound is on the displacement, not the gradient).
"""
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

import ee_oracle as O
from helpers import GOLD_DIR

pytestmark = pytest.mark.gpu


def _tensors(rng, shapes):
    return {f"t{i}": rng.normal(size=s) for i, s in enumerate(shapes)}


@pytest.mark.parametrize("kind", ["sgd", "adam"])
@pytest.mark.parametrize("gdtype", ["fp32", "bf16"])
def test_optimizer_kernel_matches_reference_update(kind, gdtype):
    import torch
    from paper_2312_04916_b200.training import make_optimizer
    rng = np.random.default_rng(3)
    shapes = [(7,), (33, 65), (1,), (4096,), (129, 3), (2049,), (64, 64)]
    ref_p = _tensors(rng, shapes)
    dev_p = {k: torch.tensor(v, dtype=torch.float32, device="cuda") for k, v in ref_p.items()}
    ref_p = {k: dev_p[k].double().cpu().numpy() for k in ref_p}  # start from the same fp32 values
    opt = make_optimizer(kind, 3e-3)
    state = {}
    for step in range(4):
        grads = _tensors(rng, shapes)
        dg = {k: torch.tensor(v, dtype=torch.float32, device="cuda") for k, v in grads.items()}
        if gdtype == "bf16":
            dg = {k: v.bfloat16() for k, v in dg.items()}
        g64 = {k: v.double().cpu().numpy() for k, v in dg.items()}
        opt.step(dev_p, dg, 0.25)
        if kind == "sgd":
            O.sgd_step(ref_p, g64, 0.25, 3e-3)
        else:
            O.adam_step(ref_p, g64, 0.25, state, 3e-3)
    torch.cuda.synchronize()
    for k in ref_p:
        ours = dev_p[k].double().cpu().numpy()
        err = np.abs(ours - ref_p[k]).max() / np.abs(ref_p[k]).max()
        assert err < 1e-5, (k, err)


def test_optimizer_rejects_bad_inputs():
    import torch
    from paper_2312_04916_b200.errors import ShapeError
    from paper_2312_04916_b200.training import Adam
    p = {"a": torch.zeros(4, device="cuda")}
    with pytest.raises(ShapeError):
        Adam(1e-3).step(p, {"a": torch.zeros(5, device="cuda")}, 1.0)
    with pytest.raises(ShapeError):
        Adam(1e-3).step({"a": torch.zeros(4, device="cuda", dtype=torch.bfloat16)},
                        {"a": torch.zeros(4, device="cuda")}, 1.0)


class _Batches:
    def __init__(self, batches):
        self.batches = batches

    def batch(self, rows, row_len, step):
        b = self.batches[step]
        assert b.shape == (rows, row_len)
        return b


def test_train_three_adam_steps_match_reference(tmp_path):
    import torch
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model
    from paper_2312_04916_b200.pipeline import WeightSchedule
    from paper_2312_04916_b200.training import train
    with open(os.path.join(GOLD_DIR, "trained.json")) as f:
        g = json.load(f)
    arr = dict(np.load(os.path.join(GOLD_DIR, "trained.npz")))
    cfg = ModelConfig(4, 64, 4, 128, 64, exits=(ExitSpec(1, "minimalistic", 0.25),
                                                 ExitSpec(2, "minimalistic", 0.5)))
    rc = SimpleNamespace(model=cfg, seed=0, stages=2, microbatch_size=2, global_batch_size=8,
                         steps=3, optimizer="adam", learning_rate=3e-3, data_seq_len=32,
                         defer_exit_forward=True, fill_bubbles=False,
                         weight_schedule=lambda: WeightSchedule("constant", early=(0.25, 0.5)))
    metrics = tmp_path / "m.jsonl"
    model, hist = train(rc, _Batches(arr["adam3_batches"]), metrics_path=str(metrics))
    lines = [json.loads(l) for l in open(metrics)]
    assert lines[0]["record"] == "header" and lines[0]["heads"] == ["exit_l1", "exit_l2", "final"]
    assert len(lines) == 4
    for ours, ref in zip(hist, g["adam3_losses"]):
        for k, v in ref.items():
            assert ours["losses"][k] == pytest.approx(v, rel=2e-2), (ours["step"], k)
    init = build_model(cfg, 0)
    for name in ("tok_emb", "layer1.wq", "layer2.w1", "final.out", "exit_l1.out"):
        ref = arr[f"adam3::{name}"]
        ours = model.params[name].data.double().cpu().numpy()
        disp = np.linalg.norm(ref - init.params[name].data)
        err = np.linalg.norm(ours - ref)
        print(f"{name}: |ours - ref| / |ref - init| = {err / disp:.4f}")
        assert err < 0.1 * disp, (name, err / disp)


class _StepBatches:
    """Replays the batches the reference's corpus served, regular (step) and
    fill (step + 10**9) draws."""

    def __init__(self, regular, fill):
        self.regular, self.fill = regular, fill

    def batch(self, rows, row_len, step):
        src = self.fill[step - 10**9] if step >= 10**9 else self.regular[step]
        assert src.shape == (rows, row_len)
        return src


def test_train_with_bubble_filling_matches_reference():
    """`train` with fill_bubbles on a 4-stage model (3 Adam steps): per-step
    per-exit losses within 2e-2 of the reference's `train` and the same
    microbatch count (4 regular + 1 Part-1 + 2 Part-2 per step;
    tests/golden/make_fill.py)."""
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    from paper_2312_04916_b200.pipeline import WeightSchedule
    from paper_2312_04916_b200.training import train
    with open(os.path.join(GOLD_DIR, "fill.json")) as f:
        g = json.load(f)["train"]
    arr = np.load(os.path.join(GOLD_DIR, "fill.npz"))
    L, h, nh, V, s_max = g["config"]
    cfg = ModelConfig(L, h, nh, V, s_max,
                      exits=tuple(ExitSpec(l, "minimalistic", w) for l, w in g["exits"]))
    rc = SimpleNamespace(model=cfg, seed=0, stages=g["stages"], microbatch_size=2,
                         global_batch_size=8, steps=g["steps"], optimizer="adam",
                         learning_rate=g["lr"], data_seq_len=32, defer_exit_forward=True,
                         fill_bubbles=True, fill_f_over_b=g["f_over_b"],
                         weight_schedule=lambda: WeightSchedule(
                             "constant", early=tuple(w for _, w in g["exits"])))
    _, hist = train(rc, _StepBatches(arr["train_batches"], arr["train_fill_batches"]))
    assert [r["microbatches"] for r in hist] == g["microbatches"]
    for ours, ref in zip(hist, g["losses"]):
        for k, v in ref.items():
            assert ours["losses"][k] == pytest.approx(v, rel=2e-2), (ours["step"], k)
