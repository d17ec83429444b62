"""Reference-side backend: the reference package's inference entry points run
on this package's sm_100a engine.

The reference chooses its numeric kernels in `eepipe/kernels.py:13-27`
(``EEPIPE_BACKEND=auto|compiled|python``).  Its inference hot path
(`eepipe/inference.py:256-539`) does not go through that selector -- it calls
the kernels per row on numpy arrays -- so the drop-in boundary is one level
up: a reference caller hands its own `EarlyExitModel` / `StagePartition`
to the functions below, which take the reference's arguments, raise the
reference's exception types and return a trace with the reference's fields.
INTEGRATION.md shows the four lines a maintainer adds to
`eepipe/inference.py` to dispatch on ``EEPIPE_BACKEND=b200``.

Everything here is conversion: the parameters are read through the
reference model's ``named_arrays()`` (`eepipe/model.py:101-102`), wrapped by
`model.model_from_arrays` (names and shapes checked against this package's
draw plan, which is the reference's), and the computation is the engine in
`inference.py` (CUDA only; there is no CPU path).
"""

from __future__ import annotations

from . import inference as _inference
from .model import EarlyExitModel, ExitSpec, ModelConfig, model_from_arrays
from .model import partition as _partition


def config_from_reference(cfg) -> ModelConfig:
    """`eepipe.model.ModelConfig` -> this package's `ModelConfig` (same
    fields, same validation, `eepipe/model.py:34-71`)."""
    return ModelConfig(cfg.num_layers, cfg.hidden_dim, cfg.num_heads, cfg.vocab_size,
                       cfg.max_seq_len,
                       exits=tuple(ExitSpec(e.layer_index, e.head_kind, e.loss_weight)
                                   for e in cfg.exits),
                       tie_embeddings=cfg.tie_embeddings)


def model_from_reference(ref_model):
    """A reference `EarlyExitModel` (float64 parameters) as this package's
    model, parameter for parameter (no copy of the float64 arrays)."""
    return model_from_arrays(config_from_reference(ref_model.config), ref_model.named_arrays())


def _model(m):
    # already one of ours, or a reference model (anything with .config and
    # .named_arrays())
    return m if isinstance(m, EarlyExitModel) else model_from_reference(m)


def generate_kv_recompute(model, prompt, threshold, max_new_tokens, max_deferred=4, *,
                          dtype="fp32"):
    """`eepipe.inference.generate_kv_recompute` (`eepipe/inference.py:256-381`)
    on the GPU.  ``dtype="fp32"`` (default) is the parity mode: identical
    tokens and exit layers to the reference; ``"bf16"`` is the performance
    path (tiled bf16 weights, TMA GEMVs)."""
    return _inference.generate_kv_recompute(_model(model), prompt, threshold, max_new_tokens,
                                            max_deferred, dtype=dtype)


def model_from_reference_partition(part):
    """The monolithic model behind a reference `StagePartition`
    (`eepipe/model.py:304-323`): every stage's parameters, tied replicas
    taken from the first stage that holds them (they are copies)."""
    arrays = {}
    for st in part.stages:
        for name, t in st.params.items():
            arrays.setdefault(name, getattr(t, "data", t))
    return model_from_arrays(config_from_reference(part.config), arrays)


def generate_pipeline(part, prompt, threshold, max_new_tokens, stage_times=None, *,
                      dtype="fp32"):
    """`eepipe.inference.generate_pipeline(part, prompt, threshold,
    max_new_tokens, stage_times)` (`eepipe/inference.py:466-539`) on the GPU.
    ``part`` is the reference's `StagePartition`; its stage layout is a pure
    function of (model, num_stages) (`eepipe/model.py:336-376`), so the bridge
    rebuilds the model and re-partitions it into the same stages."""
    model = model_from_reference_partition(part)
    return _inference.generate_pipeline(_partition(model, part.num_stages), prompt, threshold,
                                        max_new_tokens, stage_times, dtype=dtype)


def greedy_reference(model, prompt, max_new_tokens, *, dtype="fp32"):
    """`eepipe.inference.greedy_reference` (`eepipe/inference.py:547-569`)."""
    return _inference.greedy_reference(_model(model), prompt, max_new_tokens, dtype=dtype)
