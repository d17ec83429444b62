"""Distributed pipeline-based inference protocol (pipeline_infer.py) on CPU
with gloo, world sizes 2 and 4: FIFO per stage, emit-once semantics, the
status drain of stages behind the emitting one, confidence gathering and the
modeled latency — against a sequential simulation of the same stand-in
stage math (the GPU stage math itself is covered by tests/test_gpu_parity.py).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition

V = 97


def _fire(tap, pos):
    return (pos + tap) % 3 == 0


def _token(tap, pos):
    return (pos * 7 + tap * 5) % V


class FakeStage:
    """rows += 1 per local layer; head at tap t on decide position p
    fires iff (p + t) % 3 == 0 and proposes token (7p + 5t) % V."""

    def __init__(self, spec, cfg, thr):
        self.spec, self.cfg = spec, cfg
        self.device = torch.device("cpu")
        self.x_dtype = torch.float64
        self.filled = set()

    def embed(self, tokens, positions):
        return torch.tensor([[float(t)] * self.cfg.hidden_dim for t in tokens], dtype=torch.float64)

    def process(self, rows, positions, decide):
        evals = []
        heads_at = {}
        for local, hd in self.spec.heads:
            heads_at.setdefault(local, []).append(hd)
        x = rows.clone()
        for local in range(0, len(self.spec.layer_indices) + 1):
            if local > 0:
                x = x + 1
                for p in positions:
                    assert (local, p) not in self.filled
                    self.filled.add((local, p))
            if decide in positions:
                for hd in heads_at.get(local, []):
                    fired = _fire(hd.layer_index, decide) or hd.is_final
                    evals.append((hd.key, hd.layer_index, fired, _token(hd.layer_index, decide),
                                  float(decide + hd.layer_index)))
        return x, evals

    def kv_complete(self, upto):
        return all((l, p) in self.filled for l in range(1, len(self.spec.layer_indices) + 1)
                   for p in range(upto))


def _simulate(model, prompt, n_new):
    heads = sorted(model.heads, key=lambda hd: (hd.layer_index, hd.is_final))
    toks, layers = [], []
    pos = len(prompt) - 1
    for _ in range(n_new):
        for hd in heads:
            if _fire(hd.layer_index, pos) or hd.is_final:
                toks.append(_token(hd.layer_index, pos))
                layers.append(hd.layer_index)
                break
        pos += 1
    return toks, layers


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_04916_b200.pipeline_infer import generate_pipeline_dist
        cfg = ModelConfig(8, 8, 2, V, 64, exits=(ExitSpec(2, loss_weight=0.3),
                                                 ExitSpec(4, loss_weight=0.6)))
        part = partition(build_model(cfg, 0), world)
        tr = generate_pipeline_dist(part, [3, 1, 4, 1, 5], 0.5, 12,
                                    stage_factory=lambda s, c, t: FakeStage(s, c, t))
        q.put((rank, None if tr is None else (tr.tokens, tr.exit_layers, tr.exit_stages,
                                              tr.confidences, tr.total_latency)))
    except BaseException as exc:  # pragma: no cover
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_pipeline_inference_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + int(np.random.default_rng().integers(0, 2000))
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        assert not isinstance(v, str), v
    tokens, layers, stages, confs, total = res[0]
    cfg = ModelConfig(8, 8, 2, V, 64, exits=(ExitSpec(2, loss_weight=0.3),
                                             ExitSpec(4, loss_weight=0.6)))
    model = build_model(cfg, 0)
    ref_t, ref_l = _simulate(model, [3, 1, 4, 1, 5], 12)
    assert tokens == ref_t
    assert layers == ref_l
    from paper_2312_04916_b200.model import exit_stage_index
    assert stages == [exit_stage_index(l, 8, world) for l in layers]
    # every head's confidence on the decide row is logged once per token
    assert all(set(c) == {"exit_l2", "exit_l4", "final"} for c in confs)
    assert total > 0
