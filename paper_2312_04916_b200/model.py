"""Early-exit GPT: configuration, deterministic initialisation, stage partition.

Mirrors the reference model surface (`eepipe/model.py`) so a caller of the
reference finds the same names, argument meaning and errors:

* `ExitSpec`, `ModelConfig` with the same validation (`eepipe/model.py:34-71`);
* `HeadDesc`, `EarlyExitModel`, `HEAD_KINDS` (`eepipe/model.py:31`, `74-102`);
* `build_model(config, seed)` with the reference's numpy draw order
  (`eepipe/model.py:143-204`), so random-init weights are bit-identical to the
  oracle's before they are cast to the device dtype;
* `exit_stage_index`, `partition`, `StageSpec`, `StagePartition`
  (`eepipe/model.py:288-376`).

Parameters live on the host as float64 numpy arrays when drawn with the
reference order (``init="host"``; the parity path), or directly on the GPU in
the compute dtype (``init="device"``; full-size synthetic models such as the
7B/13B/30B configs, whose float64 host copy would not fit in host RAM).  The
inference engine (`inference.py`) and the training code (`training.py`) pack
these into their own HBM layouts.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

HEAD_KINDS = ("minimalistic", "norm+embed", "mlp+embed", "layer+embed")

INIT_STD = 0.02
NORM_EPS = 1e-6


@dataclass(frozen=True)
class ExitSpec:
    layer_index: int
    head_kind: str = "minimalistic"
    loss_weight: float = 1.0


@dataclass(frozen=True)
class ModelConfig:
    num_layers: int
    hidden_dim: int
    num_heads: int
    vocab_size: int
    max_seq_len: int
    exits: tuple = ()
    tie_embeddings: bool = False

    def __post_init__(self):
        # Same rules and messages as eepipe/model.py:51-71.
        object.__setattr__(self, "exits", tuple(self.exits))
        if min(self.num_layers, self.hidden_dim, self.vocab_size) <= 0:
            raise ConfigError("model dimensions must be positive")
        if self.max_seq_len <= 0 or self.num_heads <= 0:
            raise ConfigError("model dimensions must be positive")
        if self.hidden_dim % self.num_heads:
            raise ConfigError(
                f"hidden_dim {self.hidden_dim} not divisible by {self.num_heads} heads")
        taken = set()
        for spec in self.exits:
            if not 0 <= spec.layer_index <= self.num_layers:
                raise ConfigError(f"exit layer index {spec.layer_index} out of range")
            if spec.layer_index in taken:
                raise ConfigError(f"duplicate exit layer index {spec.layer_index}")
            if spec.head_kind not in HEAD_KINDS:
                raise ConfigError(f"unknown head kind {spec.head_kind!r}")
            if spec.loss_weight < 0:
                raise ConfigError("exit loss weights must be non-negative")
            taken.add(spec.layer_index)

    @property
    def head_dim(self):
        return self.hidden_dim // self.num_heads


@dataclass(frozen=True)
class HeadDesc:
    """One output head: an early exit or the final head."""

    key: str
    kind: str
    layer_index: int
    loss_weight: float
    is_final: bool
    param_names: dict = field(default_factory=dict)


class Param:
    """Holder with a ``.data`` attribute, like the reference `Tensor`
    (`eepipe/autodiff.py:35-46`): numpy float64 for host-drawn weights or a
    torch tensor for device-drawn ones."""

    __slots__ = ("data",)

    def __init__(self, data):
        self.data = data

    @property
    def shape(self):
        return tuple(self.data.shape)


class EarlyExitModel:
    """Parameters plus head layout (`eepipe/model.py:86-102`)."""

    def __init__(self, config: ModelConfig, params: dict, heads: list):
        self.config = config
        self.params = params  # canonical name -> Param, each exactly once
        self.heads = heads  # sorted by (tap, is_final)

    @property
    def early_heads(self):
        return [h for h in self.heads if not h.is_final]

    @property
    def on_device(self):
        return not isinstance(next(iter(self.params.values())).data, np.ndarray)

    def param_count(self):
        total = 0
        for p in self.params.values():
            total += int(np.prod(p.shape))
        return total

    def named_arrays(self):
        return {name: p.data for name, p in self.params.items()}


def _head_param_names(key, kind, out_name):
    names = {"out": out_name}
    if kind != "minimalistic":
        names["norm"] = f"{key}.norm"
    if kind == "mlp+embed":
        names.update(pre_norm=f"{key}.pre_norm", w1=f"{key}.w1", w2=f"{key}.w2")
    if kind == "layer+embed":
        for w in ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "w1", "w2"):
            names[w] = f"{key}.{w}"
    return names


def head_param_size(kind, hidden_dim, vocab_size, tied):
    """Parameters one exit head owns (`eepipe/model.py:120-129`)."""
    h, v = hidden_dim, vocab_size
    size = 0 if tied else v * h
    if kind != "minimalistic":
        size += h
    if kind == "mlp+embed":
        size += h + 8 * h * h
    if kind == "layer+embed":
        size += 2 * h + 12 * h * h
    return size


def expected_param_count(config: ModelConfig):
    """Closed-form parameter count (`eepipe/model.py:132-140`)."""
    h, v = config.hidden_dim, config.vocab_size
    backbone = v * h + config.max_seq_len * h + config.num_layers * (12 * h * h + 2 * h)
    final = h + v * h
    exits = sum(head_param_size(e.head_kind, h, v, config.tie_embeddings)
                for e in config.exits)
    return backbone + final + exits


def _draw_plan(config: ModelConfig):
    """The reference's parameter creation order as (name, shape, kind) with
    kind 'normal' (one N(0, 0.02) draw) or 'ones' (no draw).  Follows
    `eepipe/model.py:159-202`: embeddings, layers 1..L, final head, then exit
    heads by ascending tap.  Returns (plan, heads)."""
    h, v = config.hidden_dim, config.vocab_size
    plan = [("tok_emb", (v, h), "normal"), ("pos_emb", (config.max_seq_len, h), "normal")]
    for i in range(1, config.num_layers + 1):
        p = f"layer{i}"
        plan.append((f"{p}.attn_norm", (h,), "ones"))
        for w in ("wq", "wk", "wv", "wo"):
            plan.append((f"{p}.{w}", (h, h), "normal"))
        plan.append((f"{p}.mlp_norm", (h,), "ones"))
        plan.append((f"{p}.w1", (h, 4 * h), "normal"))
        plan.append((f"{p}.w2", (4 * h, h), "normal"))
    plan.append(("final.norm", (h,), "ones"))
    plan.append(("final.out", (v, h), "normal"))

    heads = []
    for spec in sorted(config.exits, key=lambda e: e.layer_index):
        key = f"exit_l{spec.layer_index}"
        tied = config.tie_embeddings
        names = _head_param_names(key, spec.head_kind, "tok_emb" if tied else f"{key}.out")
        if not tied:
            plan.append((names["out"], (v, h), "normal"))
        if "norm" in names:
            plan.append((names["norm"], (h,), "ones"))
        if spec.head_kind == "mlp+embed":
            plan.append((names["pre_norm"], (h,), "ones"))
            plan.append((names["w1"], (h, 4 * h), "normal"))
            plan.append((names["w2"], (4 * h, h), "normal"))
        if spec.head_kind == "layer+embed":
            plan.append((names["attn_norm"], (h,), "ones"))
            for w in ("wq", "wk", "wv", "wo"):
                plan.append((names[w], (h, h), "normal"))
            plan.append((names["mlp_norm"], (h,), "ones"))
            plan.append((names["w1"], (h, 4 * h), "normal"))
            plan.append((names["w2"], (4 * h, h), "normal"))
        heads.append(HeadDesc(key, spec.head_kind, spec.layer_index,
                              spec.loss_weight, False, names))
    heads.append(HeadDesc("final", "norm+embed", config.num_layers, 1.0, True,
                          {"norm": "final.norm", "out": "final.out"}))
    heads.sort(key=lambda hd: (hd.layer_index, hd.is_final))
    return plan, heads


def build_model(config: ModelConfig, seed: int, *, init: str = "host",
                dtype=None, device=None) -> EarlyExitModel:
    """Deterministic initialisation.

    ``init="host"`` reproduces the reference exactly: numpy
    ``default_rng(seed)`` float64 draws in the reference order
    (`eepipe/model.py:143-204`), so the same (config, seed) gives the same
    bits as `eepipe.model.build_model`.

    ``init="device"`` draws N(0, 0.02) with a seeded torch generator straight
    into ``dtype`` on ``device`` (default bf16 on cuda:0).  The values differ
    from the reference's (different generator) but the distribution and the
    structure match; this is how full-size synthetic benchmark models are
    made without a 58 GB float64 host copy.
    """
    plan, heads = _draw_plan(config)
    params = {}
    if init == "host":
        rng = np.random.default_rng(seed)
        for name, shape, kind in plan:
            if kind == "normal":
                params[name] = Param(rng.normal(0.0, INIT_STD, shape))
            else:
                params[name] = Param(np.ones(shape))
    elif init == "device":
        import torch
        dev = torch.device(device or "cuda:0")
        dt = dtype or torch.bfloat16
        gen = torch.Generator(device=dev)
        gen.manual_seed(int(seed))
        for name, shape, kind in plan:
            if kind == "normal":
                t = torch.empty(shape, dtype=dt, device=dev)
                t.normal_(0.0, INIT_STD, generator=gen)
            else:
                t = torch.ones(shape, dtype=dt, device=dev)
            params[name] = Param(t)
    else:
        raise ConfigError(f"unknown init {init!r} (expected 'host' or 'device')")
    return EarlyExitModel(config, params, heads)


def model_from_arrays(config: ModelConfig, arrays: dict) -> EarlyExitModel:
    """Wrap externally produced weights (e.g. a reference model's
    ``named_arrays()`` or a reference checkpoint) with this package's head
    layout.  Names and shapes must match `build_model`'s."""
    plan, heads = _draw_plan(config)
    params = {}
    for name, shape, _ in plan:
        if name not in arrays:
            raise ConfigError(f"missing parameter {name}")
        arr = arrays[name]
        if not isinstance(arr, np.ndarray):  # a reference Tensor / Param (ndarray.data is a buffer)
            arr = getattr(arr, "data", arr)
        if tuple(arr.shape) != tuple(shape):
            raise ConfigError(f"parameter {name} has shape {tuple(arr.shape)}, expected {shape}")
        params[name] = Param(arr)
    return EarlyExitModel(config, params, heads)


# ---------------------------------------------------------------------------
# Pipeline partition (eepipe/model.py:288-376)
# ---------------------------------------------------------------------------


@dataclass
class StageSpec:
    """Everything one pipeline stage owns; ``heads`` pairs each local head
    with the number of local layers applied before its tap."""

    index: int
    layer_indices: list
    has_embedding: bool
    heads: list  # (local_pos, HeadDesc)
    params: dict  # name -> Param (stage-local copies)


@dataclass
class StagePartition:
    config: ModelConfig
    num_stages: int
    stages: list
    tied_replicas: dict  # canonical name -> stage indices holding a copy

    def exit_stages(self):
        """Stage index of every early-exit head, in depth order."""
        return [st.index for st in self.stages for _, hd in st.heads if not hd.is_final]

    def stage_of_head(self, key):
        for st in self.stages:
            for _, hd in st.heads:
                if hd.key == key:
                    return st.index
        raise KeyError(key)


def exit_stage_index(layer_index: int, num_layers: int, num_stages: int) -> int:
    """Stage owning the tap at ``layer_index``: boundary taps go to the later
    stage, tap 0 to stage 1, tap L to the last (`eepipe/model.py:326-333`)."""
    per = num_layers // num_stages
    return min(layer_index // per + 1, num_stages)


def _copy(data):
    if isinstance(data, np.ndarray):
        return data.copy()
    return data.clone()


def partition(model: EarlyExitModel, num_stages: int, *, copy: bool = True) -> StagePartition:
    """Contiguous layers per stage, heads on `exit_stage_index`, stage-local
    parameter copies and the tied-replica map (`eepipe/model.py:336-376`).
    ``copy=False`` shares the arrays (used for device-resident models where a
    second copy would double HBM use; stages never write weights at
    inference)."""
    cfg = model.config
    if num_stages <= 0:
        raise ConfigError("stage count must be positive")
    if cfg.num_layers % num_stages:
        raise ConfigError(f"{cfg.num_layers} layers not divisible into {num_stages} stages")
    per = cfg.num_layers // num_stages
    by_stage = {s: [] for s in range(1, num_stages + 1)}
    for hd in model.heads:
        s = exit_stage_index(hd.layer_index, cfg.num_layers, num_stages)
        by_stage[s].append((hd.layer_index - (s - 1) * per, hd))
    for lst in by_stage.values():
        lst.sort(key=lambda t: (t[0], t[1].is_final))

    stages = []
    for s in range(1, num_stages + 1):
        layers = list(range((s - 1) * per + 1, s * per + 1))
        names = {"tok_emb", "pos_emb"} if s == 1 else set()
        for i in layers:
            names.update(n for n in model.params if n.startswith(f"layer{i}."))
        for _, hd in by_stage[s]:
            names.update(hd.param_names.values())
        params = {n: Param(_copy(model.params[n].data) if copy else model.params[n].data)
                  for n in sorted(names)}
        stages.append(StageSpec(s, layers, s == 1, by_stage[s], params))

    holders = {}
    for st in stages:
        for n in st.params:
            holders.setdefault(n, []).append(st.index)
    tied = {n: sorted(h) for n, h in holders.items() if len(h) > 1}
    return StagePartition(cfg, num_stages, stages, tied)
