"""The MULTI-PROCESS stage code with the real kernels, on the one GPU the
pool gives: P stage processes (torch.multiprocessing, gloo default group)
all on cuda:0, driving `pipeline_infer.generate_pipeline_dist` with the real
`GpuStage` engines and `pipeline.run_stage_1f1b_dist` with the real GPU
`StageCompute`.  NCCL refuses two ranks on one device, so the `Wire`
stages device tensors through host memory; control words go over gloo
either way.  Results must equal the threaded executors (one process, stage
threads) BITWISE: tokens, exit layers, exit stages, confidences; gradients
and per-exit losses.  The reference equivalents are its stage threads
(`eepipe/pipeline.py:596-603`, `eepipe/inference.py:485-497`).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _infer_cfg():
    return ModelConfig(4, 512, 4, 256, 64, exits=(ExitSpec(1, "minimalistic", 0.3),
                                                  ExitSpec(2, "minimalistic", 0.6)))


def _infer_worker(rank, world, port, dtype, thr, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_04916_b200.pipeline_infer import generate_pipeline_dist
        model = build_model(_infer_cfg(), 11)
        part = partition(model, world)
        prompt = [int(t) for t in np.random.default_rng(4).integers(0, 256, size=7)]
        tr = generate_pipeline_dist(part, prompt, thr, 16, dtype=dtype)
        if rank == 0:
            q.put((tr.tokens, tr.exit_layers, tr.exit_stages, tr.confidences))
    except BaseException as e:  # surfaced by the parent
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype,world", [("fp32", 2), ("bf16", 2), ("bf16", 4)])
def test_dist_pipeline_inference_on_one_gpu_equals_threaded(dtype, world):
    from paper_2312_04916_b200 import inference as I
    model = build_model(_infer_cfg(), 11)
    part = partition(model, world)
    prompt = [int(t) for t in np.random.default_rng(4).integers(0, 256, size=7)]
    for thr in (1.0, 0.99 / 256, 1.5 / 256):
        ref = I.generate_pipeline(part, prompt, thr, 16, dtype=dtype)
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _port()
        procs = [ctx.Process(target=_infer_worker, args=(r, world, port, dtype, thr, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        got = q.get(timeout=600)
        for p in procs:
            p.join(timeout=120)
        assert not isinstance(got, str), got
        tokens, layers, stages, confs = got
        assert tokens == ref.tokens, thr
        assert layers == ref.exit_layers, thr
        assert stages == ref.exit_stages, thr
        assert confs == ref.confidences, thr
        assert all(p.exitcode == 0 for p in procs)



def _train_setup(layers, exits, tie, seed):
    cfg = ModelConfig(layers, 32, 4, 64, 16, exits=exits, tie_embeddings=tie)
    model = build_model(cfg, seed)
    batch = np.random.default_rng(seed + 1000).integers(0, 64, size=(8, 9))
    return model, batch


TRAIN_CONFIGS = [
    (4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), False, 2),
    (4, (ExitSpec(1, loss_weight=0.25), ExitSpec(2, loss_weight=0.5)), True, 2),
    (8, (ExitSpec(2, loss_weight=0.25), ExitSpec(4, "mlp+embed", 0.5),
         ExitSpec(8, loss_weight=0.1)), False, 4),
]


def _train_worker(rank, world, port, cfg_idx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_04916_b200.pipeline import IterationOptions, run_stage_1f1b_dist
        layers, exits, tie, _ = TRAIN_CONFIGS[cfg_idx]
        model, batch = _train_setup(layers, exits, tie, layers * 10 + world)
        part = partition(model, world)
        grads, rep = run_stage_1f1b_dist(part, batch, IterationOptions(microbatch_size=2),
                                         model=model)
        q.put((rank, {k: v.detach().float().cpu().numpy() for k, v in grads.items()},
               dict(rep.per_exit_losses)))
    except BaseException as e:
        q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_idx", range(len(TRAIN_CONFIGS)))
def test_dist_1f1b_on_one_gpu_equals_threaded(cfg_idx):
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    layers, exits, tie, world = TRAIN_CONFIGS[cfg_idx]
    model, batch = _train_setup(layers, exits, tie, layers * 10 + world)
    part = partition(model, world)
    ref, ref_rep = run_iteration_1f1b(part, batch, IterationOptions(microbatch_size=2),
                                      model=model)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_train_worker, args=(r, world, port, cfg_idx, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    merged, losses = {}, {}
    for rank, g, lo in sorted(results, key=lambda r: r[0]):
        assert not isinstance(g, str), g
        for k, v in g.items():
            if k in merged:  # tied replica: every holder carries the all-reduced sum
                assert np.array_equal(merged[k], v), k
            merged[k] = v
        losses.update(lo)
    assert set(merged) == set(ref)
    for k, v in ref.items():
        assert np.array_equal(merged[k], v.detach().float().cpu().numpy()), k
    for k, v in ref_rep.per_exit_losses.items():
        assert losses[k] == v, k
