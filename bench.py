"""Benchmark: EE-GPT 7B early-exit decode with KV recomputation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--threshold T]
    python bench.py --impl reference ...      # the reference CPU path (oracle port)

Workload (BASELINE.json configs[2]): L=32, h=4096, nh=32,
V=50304, s_max=2048, minimalistic exits at layers 8 (w 0.1) and 16 (w 0.2),
bf16 weights/KV, batch 1, prompt 64 tokens, 256 new tokens per step,
max_deferred 4.  A "step" is one `generate_kv_recompute` call (prefill +
256 decoded tokens).  Weights are random-init N(0, 0.02) drawn on the device
(seeded torch generator; the reference's numpy draw order is used only by
the parity tests — a float64 host copy of 7B would need 58 GB).  Prompts are
`default_rng(1).integers(0, V, 64)`.  Weights (14.5 GB) exceed L2 (126 MB),
so no flush is needed between steps.

metric: decode tokens/s (whole job); `sweep` adds tokens/s, mean exit layer
and modeled speedup at every threshold of 0.2..1.0.  `roofline` is for the
dominant kernel chain, `ee_decode_layers` over all 32 layers for one row
(one launch = the full-depth KV-recompute pass), timed with CUDA events on
its stream: algorithmic bytes = 32 x (12 h^2 + 2h) x 2 B weights + K/V
write/read.  Multi-GPU: the path does not shard (one model per
GPU), so N GPUs run N independent replicas ("replicas only").
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C3 = dict(num_layers=32, hidden_dim=4096, num_heads=32, vocab_size=50304, max_seq_len=2048)
EXITS = ((8, 0.1), (16, 0.2))
PROMPT_LEN, NEW_TOKENS, MAX_DEFERRED = 64, 256, 4
SWEEP = (0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0)
METRIC = "EE-7B decode tokens/s (KV recompute, threshold sweep 0.2-1.0)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def c3_config():
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    return ModelConfig(**C3, exits=tuple(ExitSpec(l, "minimalistic", w) for l, w in EXITS))


def prompt_tokens():
    import numpy as np
    return [int(t) for t in np.random.default_rng(1).integers(0, C3["vocab_size"], PROMPT_LEN)]


def measured_traffic(ctx):
    """dram bytes (read + write) of one full-depth decode pass at the bench's
    context from the committed ncu launch list
    (profiles/r2_decode_pass_traffic.json, made by tools/decode_traffic.py
    from `ncu ... python tools/prof_decode.py 1 1 <ctx>`), next to that
    pass's algorithmic bytes."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_decode_pass_traffic.json")) as f:
            t = json.load(f)
        return {"bytes": t["traffic_bytes"], "algorithmic_bytes": t["algorithmic_bytes"],
                "ratio": t["ratio"], "ctx": t["ctx"], "same_ctx": t["ctx"] == ctx,
                "source": "profiles/r2_decode_pass_traffic.json (ncu launch list, cold cache)"}
    except Exception:
        return None


def head_traffic():
    """dram bytes (read + write) of one fused train-head call (all its
    kernels) from the committed ncu launch list, next to the minimum
    (X, W read once, dW read-modify-write, G written and read twice)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_train_head_traffic.json")) as f:
            t = json.load(f)
        return {"bytes": t["traffic_bytes"], "kernels": t["kernels"],
                "source": "profiles/r2_train_head_traffic.json (ncu)"}
    except Exception:
        return None


def decode_pass_bytes(h, L, ctx):
    """Algorithmic bytes of one full-depth single-row pass:
    weights once + K/V write of the row + K/V read of the prefix (bf16)."""
    weights = L * (12 * h * h) * 2 + L * 2 * h * 4  # bf16 matrices, fp32 norms
    kv = L * (2 * h * 2 + 2 * (ctx + 1) * h * 2)
    return weights + kv


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the REAL reference (`eepipe`, installed
# unmodified into baseline/_ref) on the host cores
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_reference(backend):
    """Import the reference package from baseline/_ref with EEPIPE_BACKEND
    set (it is read once at import, eepipe/kernels.py:13)."""
    os.environ["EEPIPE_BACKEND"] = backend
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import eepipe.kernels as k
    if k.BACKEND != backend:
        raise RuntimeError(f"reference backend {backend!r} requested, got {k.BACKEND!r}")
    import eepipe.inference as inf
    import eepipe.model as mdl
    return inf, mdl, k


class RefDecodeSlice:
    """The reference's own decode kernels on a 7B-width slice (h=4096, 32
    heads, V=50304): `_InferParams` (which pre-transposes the head matrix,
    eepipe/inference.py:147-171), `_layer_step` (216-229) on one row at the
    C3 run's mean context (prompt 64 + 128), and `head_logits` (173-185) on
    one row.  Weights from the reference's `build_model(cfg, 0)`."""

    def __init__(self, backend):
        inf, mdl, k = _import_reference(backend)
        h, V, nh = C3["hidden_dim"], C3["vocab_size"], C3["num_heads"]
        cfg = mdl.ModelConfig(1, h, nh, V, C3["max_seq_len"], exits=())
        model = mdl.build_model(cfg, 0)
        self.inf, self.backend = inf, k.BACKEND
        self.ip = inf._InferParams(model.params, model.heads, cfg, [1], True)
        self.cache = inf.KVCache([1], C3["max_seq_len"], nh, h // nh)
        rng = np.random.default_rng(0)
        self.ctx = PROMPT_LEN + NEW_TOKENS // 2
        for p in range(self.ctx):
            self.cache.fill(1, p, rng.normal(size=(nh, h // nh)), rng.normal(size=(nh, h // nh)))
        self.x = self.ip.embed([1], [self.ctx])
        self.hd, self.mats = self.ip.heads[-1]  # the final head (norm + V x h)

    def sample(self):
        """(seconds of one 1-row layer step, seconds of one head evaluation)."""
        self.cache.mask[1][self.ctx:] = False
        t0 = time.perf_counter()
        self.inf._layer_step(self.ip.layers[1], self.x, [self.ctx], self.cache, 1,
                             C3["num_heads"])
        t1 = time.perf_counter()
        self.ip.head_logits(self.hd, self.mats, self.x[0])
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1


def ref_step_seconds(t_row, t_head, threshold, new_tokens=NEW_TOKENS):
    """One C3 step (prompt 64 + new_tokens decoded) in the reference's KV
    recomputation, from its per-row layer and per-head costs.  Exact
    structure, not a model of it: every (position, layer) pair is computed
    exactly once (a deferred row later runs only the layers it skipped,
    eepipe/inference.py:316-322, 355-360), the reference's `dot_rows`
    (einsum optimize=False) costs the same per row whatever the pass width
    (measured: 5 rows = 4.9 x 1 row), so layer time = rows x 32 x t_row with
    rows = 64 prompt + new_tokens; head evaluations: threshold 1.0 evaluates
    all 3 heads for every decided token (inference.py:293-311); below 1.0 at
    least the first head is evaluated, and 1 per token is used (the lower
    bound, i.e. the FASTEST the reference can be at that threshold)."""
    L = C3["num_layers"]
    heads = 3 if threshold >= 1.0 else 1
    rows = PROMPT_LEN + new_tokens
    return rows * L * t_row + (new_tokens + 1) * heads * t_head


def _cpu_info():
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"os_cpu_count": os.cpu_count(), "affinity_cpus": aff}


def reference_decode_baseline(threshold, samples=3, compiled=True):
    """Both reference backends on the host: numpy (`EEPIPE_BACKEND=python`,
    in process) and Cython (`compiled`, in a subprocess since the backend is
    fixed at import).  Returns the faster backend's tokens/s at C3 plus the
    per-op timings of both."""
    sl = RefDecodeSlice("python")
    sl.sample()
    ts = [sl.sample() for _ in range(samples)]
    t_row = float(np.median([t[0] for t in ts]))
    t_head = float(np.median([t[1] for t in ts]))
    res = {"python": {"layer_row_s": t_row, "head_s": t_head, "samples": samples}}
    if compiled:
        try:
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-probe",
                                  "compiled"], capture_output=True, text=True, timeout=240)
            res["compiled"] = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception as e:  # report, never fall back to our code
            res["compiled"] = {"error": str(e)[:200]}
    best = min((k for k in res if "layer_row_s" in res[k]),
               key=lambda k: ref_step_seconds(res[k]["layer_row_s"], res[k]["head_s"], threshold))
    step = ref_step_seconds(res[best]["layer_row_s"], res[best]["head_s"], threshold)
    return {"tokens_per_s": NEW_TOKENS / step, "step_s": step, "backend": best,
            "per_backend": res, "ctx": sl.ctx}


def ref_probe(backend):
    sl = RefDecodeSlice(backend)
    t_row, t_head = sl.sample()
    print(json.dumps({"layer_row_s": t_row, "head_s": t_head, "samples": 1}))
    return 0


def cpu_head_timing(n=256, h=2048, V=50304):
    """The reference's training exit head on the host: eepipe autodiff
    `matmul(x, out, transpose_b=True)` -> `cross_entropy` -> `backward`
    (eepipe/model.py:219-230, autodiff.py:158-179, 301-323; numpy `@` on
    OpenBLAS with all host threads) on an n-row slice of the C2 shape,
    GFLOP/s on the same 6 n h V count as the GPU number."""
    _import_reference(os.environ.get("EEPIPE_BACKEND", "python"))
    from eepipe import autodiff as ad
    rng = np.random.default_rng(0)
    x = ad.Tensor(rng.normal(size=(n, h)), requires_grad=True)
    w = ad.Tensor(rng.normal(0, 0.02, size=(V, h)), requires_grad=True)
    t = rng.integers(0, V, size=n)

    def run(rows):
        with ad.Tape():
            loss = ad.cross_entropy(ad.matmul(x if rows == n else ad.Tensor(x.data[:rows],
                                                                           requires_grad=True),
                                              w, transpose_b=True), t[:rows])
            ad.backward(loss)
    run(8)
    t0 = time.perf_counter()
    run(n)
    dt = time.perf_counter() - t0
    return {"value": 6 * n * h * V / dt / 1e9, "unit": "GFLOP/s (6nhV)", "cores": os.cpu_count(),
            "kind": "reference", **_cpu_info(),
            "sample": f"reference eepipe autodiff (float64, numpy/OpenBLAS, backend "
                      f"{os.environ.get('EEPIPE_BACKEND')}) C2 exit head fwd+bwd on {n} of the "
                      f"4096 rows: {dt:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sl = RefDecodeSlice("python")
    for _ in range(args.warmup):
        sl.sample()
    t0 = time.perf_counter()
    ts = [sl.sample() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    t_row = float(np.median([t[0] for t in ts]))
    t_head = float(np.median([t[1] for t in ts]))
    step = ref_step_seconds(t_row, t_head, args.threshold, args.new_tokens)
    value = args.new_tokens / step
    try:
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-probe",
                              "compiled"], capture_output=True, text=True, timeout=240)
        comp = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:
        comp = {"error": str(e)[:200]}
    backend = "python"
    if "layer_row_s" in comp:
        cstep = ref_step_seconds(comp["layer_row_s"], comp["head_s"], args.threshold,
                                 args.new_tokens)
        if cstep < step:
            backend, step, value = "compiled", cstep, args.new_tokens / cstep
    sample = (f"reference eepipe (baseline/_ref, unmodified; backend {backend}: numpy "
              f"{t_row * 1e3:.0f} ms per 1-row _layer_step at ctx {sl.ctx} + {t_head * 1e3:.0f} ms "
              f"per head_logits, median of {args.steps}; Cython backend {comp}) on a 7B-width slice "
              f"(h=4096, V=50304); one C3 step = (64 prompt + {args.new_tokens} new rows) x 32 "
              f"layers x t_row + heads x t_head ({'3' if args.threshold >= 1.0 else '>=1'} per "
              f"token at threshold {args.threshold}) — the reference computes every "
              f"(position, layer) once and its per-row cost does not depend on the pass width")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "C3 EE-GPT 7B decode, KV recomputation",
                       "threshold": args.threshold, "prompt_len": PROMPT_LEN,
                       "new_tokens": args.new_tokens, "max_deferred": MAX_DEFERRED,
                       "sampled": "7B-width 1-layer slice, per-op timings composed to the C3 step"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "reference",
                             "sample": sample, **_cpu_info(),
                             "sample_wall_s": wall},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def bench_train_head(local, hbm_peak, reps=10, n=4096, h=2048, V=50304, tag="C2"):
    """Fused training exit head (loss + dX + dW, tcgen05) at a training
    shape: C2 = n 2 x 2048 tokens, h 2048; C4 = n 1 x 2048, h 5120; V = 50304,
    bf16.  TFLOP/s on the algorithmic 6 n h V, vs the measured
    bf16 peak."""
    import torch
    from paper_2312_04916_b200.training import exit_head_loss_and_grads
    _, tf_peak, kind = peaks()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            sustained = float(json.load(f).get("bf16_tflops_sustained", tf_peak))
    except Exception:
        sustained = tf_peak
    dev = f"cuda:{local}"
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(n, h, device=dev, generator=g).bfloat16()
    w = (torch.randn(V, h, device=dev, generator=g) * 0.02).bfloat16()
    t = torch.randint(0, V, (n,), device=dev, generator=g)
    acc = torch.zeros(V, h, device=dev)
    for _ in range(3):
        exit_head_loss_and_grads(x, w, t, 1.0, dw_acc=acc)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        exit_head_loss_and_grads(x, w, t, 1.0, dw_acc=acc)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    tflops = 6 * n * h * V / (ms * 1e-3) / 1e12
    return {"workload": f"{tag} exit head fwd+bwd (n={n}, h={h}, V={V}, bf16)",
            "ms": ms, "tflops_6nhv": tflops,
            "note": "executed FLOPs = algorithmic 6nhV (logits computed once: part-normalised "
                    "probabilities + in-place gradient fixup, no recompute)",
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": tf_peak,
                         "unit": "TFLOP/s", "frac": tflops / tf_peak,
                         "frac_of_sustained": tflops / sustained, "peak_kind": kind,
                         "traffic": head_traffic() if tag == "C2" else None}}


def bench_pipeline_stages(model, prompt, local, new_tokens=64, thresholds=(1.0, 0.8, 0.2)):
    """`generate_pipeline` on the C3 model at P = 2, 4, 8 stages.  The pool
    gives ONE GPU, so the stage workers are host threads with their own CUDA
    streams sharing it (the multi-process NCCL path, pipeline_infer.
    generate_pipeline_dist, is protocol-tested on gloo): all stages' layers
    still run for every token (KV fill), so throughput is bounded by the
    single GPU's full-depth rate; early exits shorten the emit latency
    (modeled speedup, eepipe/schedule.py:553-590)."""
    import torch
    from paper_2312_04916_b200 import inference as I
    from paper_2312_04916_b200.model import partition
    out = {"note": "P stage workers = threads + CUDA streams on ONE B200 (1-GPU pool); "
                   f"{new_tokens} new tokens, prompt {len(prompt)}; every stage still runs all its "
                   "layers per token (KV fill), so throughput is bounded by the single GPU's "
                   "full-depth rate, and at P=8 the eight Python stage threads of one "
                   "interpreter contend for the GIL (the multi-GPU design runs one process "
                   "per stage: pipeline_infer.generate_pipeline_dist)"}
    for P in (2, 4, 8):
        part = partition(model, P, copy=False)
        I.generate_pipeline(part, prompt, 0.8, 4, devices=[f"cuda:{local}"])  # builds stage engines
        res = {}
        for thr in thresholds:
            torch.cuda.synchronize()
            t = time.perf_counter()
            tr = I.generate_pipeline(part, prompt, thr, new_tokens, devices=[f"cuda:{local}"])
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            res[str(thr)] = {"tokens_per_s": len(tr.tokens) / dt,
                             "mean_exit_layer": tr.mean_exit_layer,
                             "modeled_speedup": tr.speedup}
        out[f"P{P}"] = res
        for spec in part.stages:  # free this partition's packed stage weights
            spec.__dict__.pop("_ee_engines", None)
        del part
        torch.cuda.empty_cache()
    return out


def bench_train_step(local, steps=3, warmup=4, M=4, mb=4, seq=2048, cfg=None, workload=None):
    """One training step: by default C2 (BASELINE configs[1]): EE-GPT 1.3B
    (L=24, h=2048, 16 heads, V=50304, tied exits at 6 (w 0.25) / 12 (w 0.5)),
    global batch 16 x 2048 as M=4 microbatches of 4 sequences (the
    microbatch split is free at P=1: 4 x 4 measured 358 ms against 377 ms for
    2 x 8 and 366 ms for 16 x 1), 1F1B executor at P=1 on 1 GPU: bf16 compute
    on the own kernels (tcgen05 CTA-pair GEMMs for every backbone linear with
    GELU / residual epilogues, tcgen05 causal attention, fused RMSNorm
    kernels, fused tcgen05 exit heads), float32 gradient accumulation in the
    weight-gradient GEMM epilogue, fused Adam on float32 master weights.  Device-drawn N(0, 0.02) weights, uniform random
    tokens.  CUDA events around whole steps (optimizer included)."""
    import torch
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition
    from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b
    from paper_2312_04916_b200.training import Adam, apply_update
    import gc
    gc.collect()
    gc.freeze()  # the decode run's host objects stay out of every GC pass of the training loop
    torch.cuda.empty_cache()
    dev = f"cuda:{local}"
    if cfg is None:
        cfg = ModelConfig(24, 2048, 16, 50304, 2048,
                          exits=(ExitSpec(6, "minimalistic", 0.25),
                                 ExitSpec(12, "minimalistic", 0.5)),
                          tie_embeddings=True)
        workload = ("C2 EE-GPT 1.3B training step (L=24, h=2048, V=50304, seq 2048, "
                    f"global batch {M * mb} x {seq} as microbatch {mb} x {M}, tied exits 6/12, "
                    "P=1, Adam, bf16 compute)")
    master = build_model(cfg, 0, init="device", dtype=torch.float32, device=dev)
    opt = Adam(3e-4)
    rng = np.random.default_rng(0)
    batches = [rng.integers(0, cfg.vocab_size, size=(M * mb, seq + 1)) for _ in range(steps + warmup)]
    part = partition(master, 1, copy=False)
    computes = []

    def step(i):
        grads, rep = run_iteration_1f1b(part, batches[i], IterationOptions(microbatch_size=mb),
                                        model=master, devices=[dev], master_dtype=torch.float32,
                                        stage_computes=computes)
        apply_update(opt, master, grads, computes, 1.0 / M)
        return rep

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        rep = step(warmup + i)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    tokens = M * mb * seq
    n_params = sum(p.data.numel() for p in master.params.values())
    h, L = cfg.hidden_dim, cfg.num_layers
    n_heads = len(master.heads)
    # model FLOPs: 6 x tokens x matmul parameters (layers + every head's h x V
    # projection) + causal attention 6 x tokens x seq x h per layer (fwd 2 S h
    # per token with the causal half, x3 for fwd + bwd)
    flops = 6 * tokens * (12 * h * h * L + n_heads * h * cfg.vocab_size) + 6 * tokens * seq * h * L
    out = {"workload": workload, "ms_per_step": ms, "tokens_per_s": tokens / (ms / 1e3),
           "tokens_per_step": tokens, "params": n_params,
           "model_tflops_per_s": flops / (ms / 1e3) / 1e12,
           "per_exit_loss": rep.per_exit_losses, "steps": steps, "warmup": warmup}
    del computes[:], master, opt
    torch.cuda.empty_cache()
    gc.unfreeze()
    return out


def bench_c4_stage(local):
    """C4 (13B, 4-stage pipeline, per-stage exits) does not fit one GPU with
    float32 master weights and Adam state (18 B/param x 13.4 B); one STAGE
    does: 10 layers at h=5120 (40 heads of 128), V=50304, microbatch 1 x
    seq 2048, M=8 microbatches, trained at P=1 with one early exit at local
    depth 5 plus the final head -- a stage's 10 layers + head, with one extra
    head (C4 stages 2-4 each own 10 layers and one head; stage 1 owns the
    embedding).  Plus the fused exit head alone at the C4 shape (n 2048,
    h 5120) vs the bf16 peak."""
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig
    cfg = ModelConfig(10, 5120, 40, 50304, 2048, exits=(ExitSpec(5, "minimalistic", 0.25),))
    out = bench_train_step(local, steps=2, warmup=2, M=8, mb=1, seq=2048, cfg=cfg,
                           workload="C4 stage slice: 10 layers, h=5120, 40 heads, V=50304, "
                                    "microbatch 1 x 8 of seq 2048, exit at 5 + final head, "
                                    "P=1, Adam, bf16 compute (1-GPU emulation of one C4 stage)")
    hbm_peak, _, _ = peaks()
    out["exit_head"] = bench_train_head(local, hbm_peak, n=2048, h=5120, tag="C4")
    return out


def bench_c5(local, new_tokens=128, pipe_tokens=32):
    """C5 (30B: L=48, h=7168, 56 heads of 128, V=50304, exits at 12 / 24)
    on ONE B200 (bf16 weights 59 GB): KV recomputation at thresholds
    1.0 / 0.8 / 0.5 / 0.2 (prompt 64, CUDA events on the engine stream), the
    full-depth one-row pass against the HBM roofline, then pipeline-based
    inference (`generate_pipeline`) at P = 2 / 4 / 8 stage threads sharing
    the GPU -- a 1-GPU emulation of the 2/4/8-stage C5 deployment."""
    import torch
    from paper_2312_04916_b200 import inference as I
    from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model
    torch.cuda.empty_cache()
    hbm_peak, _, peak_kind = peaks()
    dev = f"cuda:{local}"
    cfg = ModelConfig(48, 7168, 56, 50304, 2048,
                      exits=(ExitSpec(12, "minimalistic", 0.1), ExitSpec(24, "minimalistic", 0.2)))
    model = build_model(cfg, 0, init="device", dtype=torch.bfloat16, device=dev)
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, cfg.vocab_size, PROMPT_LEN)]
    I.generate_kv_recompute(model, prompt, 0.8, 8, MAX_DEFERRED, device=dev)  # engine build
    eng = next(iter(model.__dict__["_ee_engines"].values()))
    st = eng.stream
    sweep = {}
    for thr in (1.0, 0.8, 0.5, 0.2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        tr = I.generate_kv_recompute(model, prompt, thr, new_tokens, MAX_DEFERRED, device=dev)
        b.record(st)
        st.synchronize()
        sec = a.elapsed_time(b) / 1e3
        sweep[str(thr)] = {"tokens_per_s": len(tr.tokens) / sec,
                           "mean_exit_layer": tr.mean_exit_layer,
                           "early_exits": int(sum(1 for e in tr.exit_layers if e < cfg.num_layers)),
                           "modeled_speedup": tr.speedup}
    L, h = cfg.num_layers, cfg.hidden_dim
    ctx = PROMPT_LEN + new_tokens // 2
    with torch.cuda.device(eng.device), torch.cuda.stream(st):
        eng.kv.reset()
        eng.upload_ctrl([ctx])
        for _ in range(3):
            eng.run_layers(0, L, 1, [1] * L, ctx, 0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(10):
            eng.run_layers(0, L, 1, [1] * L, ctx, 0)
        b.record(st)
        st.synchronize()
    pass_ms = a.elapsed_time(b) / 10
    pass_bytes = decode_pass_bytes(h, L, ctx)
    achieved = pass_bytes / (pass_ms / 1e3) / 1e9
    model.__dict__.pop("_ee_engines", None)
    del eng
    torch.cuda.empty_cache()
    pipe = bench_pipeline_stages(model, prompt, local, new_tokens=pipe_tokens)
    del model
    torch.cuda.empty_cache()
    return {"workload": "C5 EE-GPT 30B (L=48, h=7168, V=50304, exits 12/24) on ONE B200, bf16, "
                        f"prompt {PROMPT_LEN}, {new_tokens} new tokens, max_deferred {MAX_DEFERRED}",
            "sweep": sweep,
            "roofline": {"bound": "hbm", "kernel": "ee_decode_layers (48 layers, 1 row)",
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "peak_kind": peak_kind, "pass_ms": pass_ms,
                         "algorithmic_bytes": pass_bytes, "ctx": ctx},
            "pipeline_stages_1gpu": pipe}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--threshold", type=float, default=0.8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train-head", action="store_true")
    ap.add_argument("--no-train-step", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--new-tokens", type=int, default=NEW_TOKENS)
    ap.add_argument("--ref-probe", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.ref_probe:
        return ref_probe(args.ref_probe)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2312_04916_b200 import inference as I
    from paper_2312_04916_b200 import _lib
    from paper_2312_04916_b200.model import build_model

    hbm_peak, _, peak_kind = peaks()
    cfg = c3_config()
    model = build_model(cfg, 0, init="device", dtype=torch.bfloat16, device=f"cuda:{local}")
    prompt = prompt_tokens()
    gen = lambda thr: I.generate_kv_recompute(model, prompt, thr, args.new_tokens, MAX_DEFERRED,
                                              device=f"cuda:{local}")
    # warm-up (builds the packed engine, touches every kernel)
    for _ in range(args.warmup):
        gen(args.threshold)
    eng = next(iter(model.__dict__["_ee_engines"].values()))
    # free the unpacked copy: the engine holds the packed layout
    stream = eng.stream

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region --------------------------------------------------------
    eng.launches = 0
    eng.h2d_bytes = eng.d2h_bytes = 0
    barrier()
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        w0 = time.perf_counter()
        traces = [gen(args.threshold) for _ in range(args.steps)]
        ev1.record(stream)
        barrier()
        wall = time.perf_counter() - w0
    dev_s = ev0.elapsed_time(ev1) / 1e3
    t = torch.tensor([dev_s, wall], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, wall = float(t[0]), float(t[1])
    tokens = sum(len(tr.tokens) for tr in traces) * world
    value = tokens / dev_s
    e2e = tokens / wall
    launches = eng.launches
    h2d, d2h = eng.h2d_bytes / args.steps, eng.d2h_bytes / args.steps
    clocks = clk.summary()

    # ---- dominant kernel chain: full-depth decode pass, 1 row ----------------
    L, h = cfg.num_layers, cfg.hidden_dim
    ctx = PROMPT_LEN + args.new_tokens // 2
    with torch.cuda.device(eng.device), torch.cuda.stream(stream):
        eng.kv.reset()
        eng.upload_ctrl([ctx])
        reps = 20
        for _ in range(3):
            eng.run_layers(0, L, 1, [1] * L, ctx, 0)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            eng.run_layers(0, L, 1, [1] * L, ctx, 0)
        b.record(stream)
        stream.synchronize()
    pass_ms = a.elapsed_time(b) / reps
    pass_bytes = decode_pass_bytes(h, L, ctx)
    achieved = pass_bytes / (pass_ms / 1e3) / 1e9

    # ---- threshold sweep --------------------------------------------------------
    sweep = {}
    if not args.no_sweep:
        for thr in SWEEP:
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            tr = gen(thr)
            s1.record(stream)
            stream.synchronize()
            sec = s0.elapsed_time(s1) / 1e3
            sweep[str(thr)] = {"tokens_per_s": len(tr.tokens) / sec,
                               "mean_exit_layer": tr.mean_exit_layer,
                               "early_exits": int(sum(1 for e in tr.exit_layers if e < L)),
                               "modeled_speedup": tr.speedup}

    # ---- pipeline-based inference: P stage workers on this one GPU ------------
    pipe = None
    if not args.no_pipeline and world == 1:
        pipe = bench_pipeline_stages(model, prompt, local)

    # ---- C5 30B on this one GPU (KV recompute sweep, pipeline P=2/4/8) ------
    c5 = None
    if not args.no_c5 and world == 1:
        model.__dict__.pop("_ee_engines", None)
        del eng, model
        torch.cuda.empty_cache()
        c5 = bench_c5(local)

    # ---- fused training exit head at the C2 shape (second half of the metric) --
    head_train = None
    if not args.no_train_head:
        head_train = bench_train_head(local, hbm_peak)
    if head_train is not None and not args.no_cpu_baseline and world == 1:
        head_train["cpu_baseline"] = cpu_head_timing()
    train_step = None
    if not args.no_train_step:
        train_step = bench_train_step(local)
    c4 = None
    if not args.no_c4 and world == 1:
        c4 = bench_c4_stage(local)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        rb = reference_decode_baseline(args.threshold)
        pb = rb["per_backend"]["python"]
        cpu = {"value": rb["tokens_per_s"], "unit": "tokens/s", "cores": 1, "kind": "reference",
               **_cpu_info(), "backend": rb["backend"], "per_backend": rb["per_backend"],
               "sample": f"reference eepipe (baseline/_ref) on a 7B-width slice: 1-row _layer_step "
                         f"{pb['layer_row_s'] * 1e3:.0f} ms at ctx {rb['ctx']} + head_logits "
                         f"{pb['head_s'] * 1e3:.0f} ms (numpy backend; Cython in per_backend), "
                         f"composed to one C3 step at threshold {args.threshold} "
                         f"(see ref_step_seconds)"}

    tr = traces[-1]
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (device-drawn N(0,0.02) weights, default_rng(1) prompt)",
        "config": {"workload": "C3 EE-GPT 7B decode, KV recomputation",
                   "layers": L, "hidden": h, "heads": cfg.num_heads, "vocab": cfg.vocab_size,
                   "exits": [list(e) for e in EXITS], "threshold": args.threshold,
                   "prompt_len": PROMPT_LEN, "new_tokens": args.new_tokens,
                   "max_deferred": MAX_DEFERRED, "batch": 1,
                   "parallelism": f"replicas x{world}",
                   "l2": "inputs larger than L2 (14.5 GB weights), no flush"},
        "mean_exit_layer": tr.mean_exit_layer,
        "early_exit_fraction": sum(1 for e in tr.exit_layers if e < L) / len(tr.exit_layers),
        "modeled_speedup": tr.speedup,
        "roofline": {"bound": "hbm", "kernel": "ee_decode_layers (32 layers, 1 row)",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                     "pass_ms": pass_ms, "algorithmic_bytes": pass_bytes,
                     "traffic": measured_traffic(ctx)},
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks,
        "sweep": sweep,
        "exit_head_train": head_train,
        "train_step": train_step,
        "pipeline_stages_1gpu": pipe,
        "c5_1gpu": c5,
        "c4_stage_1gpu": c4,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
