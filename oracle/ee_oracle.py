"""CPU oracle for the early-exit inference hot path — TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference algorithm (`eepipe`), used as the
checker in `tests/`, in `__graft_entry__.smoke()` and as the `cpu_baseline` /
`--impl reference` leg of `bench.py`.  Nothing in the product package
(`paper_2312_04916_b200/`) may import this module.

Pinned: `tests/test_oracle_golden.py` checks every function here against
golden vectors produced by the reference itself (`tests/golden/make_golden.py`
imports `/root/reference/pkg` with ``EEPIPE_BACKEND=python`` and records
tokens, exit layers, confidences and logits) — the comparison is bitwise for
the numpy backend, because this module reduces in the same order
(`np.einsum(..., optimize=False)`, `eepipe/_pykernels.py:115-121`).

Every function cites the reference lines it restates.  The oracle works on
plain dicts of float64 arrays keyed by the reference parameter names, so the
same weights can be fed to it and to the GPU engine.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

EPS = 1e-6
_INV_SQRT2 = 1.0 / math.sqrt(2.0)


class OracleError(Exception):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind  # "config" | "token" | "nonfinite"


# --- numeric kernels (eepipe/_pykernels.py) -------------------------------


def gelu(x):
    """exact erf GELU (`_pykernels.py:27-28`)."""
    return 0.5 * x * (1.0 + erf(x * _INV_SQRT2))


def rmsnorm(x, w, eps=EPS):
    """y = x / sqrt(mean(x^2) + eps) * w (`_pykernels.py:36-41`)."""
    inv = 1.0 / np.sqrt(np.mean(x * x, axis=1) + eps)
    return x * inv[:, None] * w[None, :]


def dot_rows(a, b):
    """Row-stable (m,k)@(k,n), ascending-k per element (`_pykernels.py:115-121`)."""
    return np.einsum("mk,kn->mn", a, b, optimize=False)


# --- exit decision (eepipe/inference.py:118-133) ---------------------------


def exit_decision(logits, threshold):
    z = np.asarray(logits, dtype=np.float64).ravel()
    if not np.isfinite(z).all():
        raise OracleError("nonfinite", "non-finite exit logits")
    if not (0.0 < threshold <= 1.0):
        raise OracleError("config", "threshold must lie in (0, 1]")
    e = np.exp(z - z.max())
    p = e / e.sum()
    tok = int(np.argmax(p))
    conf = float(p[tok])
    return (threshold < 1.0 and conf > threshold), tok, conf


# --- model pieces (eepipe/inference.py:141-229) ----------------------------


def head_logits(P, head, x_row):
    """One row through a head (`inference.py:175-185`).  ``head`` is a dict
    with keys kind, and the parameter names of out / norm / pre_norm / w1 / w2."""
    x = x_row[None, :]
    if head["kind"] == "mlp+embed":
        h2 = rmsnorm(x, P[head["pre_norm"]])
        x = x + dot_rows(gelu(dot_rows(h2, P[head["w1"]])), P[head["w2"]])
    if head.get("norm"):
        x = rmsnorm(x, P[head["norm"]])
    # the reference pre-transposes every head matrix once (inference.py:167)
    outT = head.get("outT")
    if outT is None:
        outT = np.ascontiguousarray(P[head["out"]].T)
    return dot_rows(x, outT)[0]


def embed(P, vocab, tokens, positions):
    """tok_emb[t] + pos_emb[p] (`inference.py:187-191`)."""
    t = np.asarray(tokens)
    if t.size and (t.min() < 0 or t.max() >= vocab):
        raise OracleError("token", "token id out of vocabulary range")
    return P["tok_emb"][t] + P["pos_emb"][np.asarray(positions)]


class KV:
    """Per-layer K/V with a monotone fill mask (`inference.py:40-73`)."""

    def __init__(self, layers, s_max, nh, dh):
        self.k = {l: np.zeros((s_max, nh, dh)) for l in layers}
        self.v = {l: np.zeros((s_max, nh, dh)) for l in layers}
        self.mask = {l: np.zeros(s_max, dtype=bool) for l in layers}

    def fill(self, l, pos, k, v):
        if self.mask[l][pos]:
            raise OracleError("config", f"KV at layer {l}, position {pos} already filled")
        self.k[l][pos], self.v[l][pos], self.mask[l][pos] = k, v, True

    def view(self, l, upto):
        if not self.mask[l][:upto].all():
            raise OracleError("config", f"reading unfilled KV at layer {l} below {upto}")
        return self.k[l][:upto], self.v[l][:upto]

    def complete(self, upto):
        return all(m[:upto].all() for m in self.mask.values())


def attend_rows(q, positions, kv, layer, nh):
    """Per-row causal attention over cache[0..pos] (`inference.py:194-213`)."""
    h = q.shape[1]
    dh = h // nh
    scale = 1.0 / np.sqrt(dh)
    out = np.empty_like(q)
    for r, pos in enumerate(positions):
        kb, vb = kv.view(layer, pos + 1)
        s = np.einsum("hd,thd->ht", q[r].reshape(nh, dh), kb, optimize=False) * scale
        e = np.exp(s - s.max(axis=1, keepdims=True))
        p = e / e.sum(axis=1, keepdims=True)
        out[r] = np.einsum("ht,thd->hd", p, vb, optimize=False).reshape(h)
    return out


def layer_step(P, l, x, positions, kv, nh):
    """One decode layer; K/V for every row are written before attending
    (`inference.py:216-229`)."""
    pre = f"layer{l}."
    h1 = rmsnorm(x, P[pre + "attn_norm"])
    q, k, v = (dot_rows(h1, P[pre + w]) for w in ("wq", "wk", "wv"))
    dh = x.shape[1] // nh
    for r, pos in enumerate(positions):
        kv.fill(l, pos, k[r].reshape(nh, dh), v[r].reshape(nh, dh))
    x = x + dot_rows(attend_rows(q, positions, kv, l, nh), P[pre + "wo"])
    h2 = rmsnorm(x, P[pre + "mlp_norm"])
    return x + dot_rows(gelu(dot_rows(h2, P[pre + "w1"])), P[pre + "w2"])


# --- generation drivers ---------------------------------------------------


class Cfg:
    def __init__(self, L, h, nh, V, s_max):
        self.L, self.h, self.nh, self.V, self.s_max = L, h, nh, V, s_max


def pretranspose(P, heads):
    """Cache each head's transposed output matrix, as `_InferParams` does
    once at construction (inference.py:167)."""
    for hd in heads:
        hd["outT"] = np.ascontiguousarray(P[hd["out"]].T)
    return heads


def heads_of(model_heads):
    """Convert HeadDesc-like objects to oracle head dicts (sorted as given)."""
    out = []
    for hd in model_heads:
        d = {"key": hd.key, "kind": hd.kind, "tap": hd.layer_index,
             "final": hd.is_final}
        d.update(hd.param_names)
        out.append(d)
    return out


def full_units(cfg, n_heads):
    """`inference.py:246-248`."""
    return cfg.L * 1.0 + 0.5 * n_heads


def generate_kv_recompute(P, cfg, heads, prompt, threshold, max_new, max_deferred=4):
    """KV-recomputation decoding (`inference.py:256-381`).  Returns a dict
    with tokens, exit_layers, confidences, latencies, total/baseline."""
    if max_deferred < 1:
        raise OracleError("config", "max_deferred must be at least 1")
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise OracleError("config", "prompt must be non-empty")
    if len(prompt) + max_new > cfg.s_max:
        raise OracleError("token", "context exceeds max_seq_len")
    L = cfg.L
    kv = KV(range(1, L + 1), cfg.s_max, cfg.nh, cfg.h // cfg.nh)
    conf = {}
    units = full_units(cfg, len(heads))

    def run_pass(xs, pos, entry, decide, forced):
        x = xs.copy()
        decision = [None]

        def tap_eval(tap):
            for hd in heads:
                if hd["tap"] != tap:
                    continue
                for r, p in enumerate(pos):
                    e = entry[r]
                    if not ((tap > e or (tap == 0 and e == 0)) and (p == decide or e > 0)):
                        continue
                    fire, tok, c = exit_decision(head_logits(P, hd, x[r]), threshold)
                    conf.setdefault(p, {})[hd["key"]] = c
                    if p == decide and decision[0] is None:
                        if hd["final"]:
                            decision[0] = (tok, L)
                        elif fire:
                            decision[0] = (tok, hd["tap"])

        tap_eval(0)
        if decision[0] is not None and not forced and decision[0][1] == 0:
            return decision[0], 0, x
        for l in range(1, L + 1):
            act = [r for r in range(len(pos)) if entry[r] < l]
            if act:
                x[act] = layer_step(P, l, x[act], [pos[r] for r in act], kv, cfg.nh)
            tap_eval(l)
            if decision[0] is not None and not forced and decision[0][1] == l and l < L:
                return decision[0], l, x
        return decision[0], L, x

    t0 = len(prompt)
    dec, _, _ = run_pass(embed(P, cfg.V, prompt, range(t0)), list(range(t0)), [0] * t0,
                         t0 - 1, True)
    depths = [L]
    tokens, exits = [], []
    deferred = []  # (position, exit_layer, hidden)
    position = t0 - 1
    for i in range(max_new):
        tokens.append(dec[0])
        exits.append(dec[1])
        if i == max_new - 1:
            break
        position += 1
        forced = len(deferred) >= max_deferred
        new = embed(P, cfg.V, [dec[0]], [position])
        xs = np.concatenate([np.stack([d[2] for d in deferred]), new]) if deferred else new
        pos = [d[0] for d in deferred] + [position]
        ent = [d[1] for d in deferred] + [0]
        dec, depth, out = run_pass(xs, pos, ent, position, forced)
        depths.append(depth)
        if depth < L:
            deferred = [(d[0], max(d[1], depth), out[r].copy()) for r, d in enumerate(deferred)]
            deferred.append((position, depth, out[-1].copy()))
        else:
            deferred = []
        assert len(deferred) <= max_deferred
    flush = 0.0
    if deferred:
        run_pass(np.stack([d[2] for d in deferred]), [d[0] for d in deferred],
                 [d[1] for d in deferred], None, True)
        flush = units
    gen = len(tokens)
    if gen and not kv.complete(t0 + gen - 1):
        raise OracleError("config", "KV fill mask incomplete after generation")
    lat = [units * d / L for d in depths[:gen]]
    return {
        "tokens": tokens, "exit_layers": exits,
        "confidences": [conf.get(t0 - 1 + i, {}) for i in range(gen)],
        "latencies": lat, "total_latency": sum(lat) + flush,
        "baseline_latency": units * gen, "pass_depths": depths,
    }


def greedy_reference(P, cfg, heads, prompt, max_new):
    """Uncached full-recompute greedy decoding with the final head
    (`inference.py:547-569`)."""
    final = [hd for hd in heads if hd["final"]][0]
    toks = [int(t) for t in prompt]
    out = []
    for _ in range(max_new):
        kv = KV(range(1, cfg.L + 1), cfg.s_max, cfg.nh, cfg.h // cfg.nh)
        pos = list(range(len(toks)))
        x = embed(P, cfg.V, toks, pos)
        for l in range(1, cfg.L + 1):
            x = layer_step(P, l, x, pos, kv, cfg.nh)
        _, tok, _ = exit_decision(head_logits(P, final, x[-1]), 1.0)
        out.append(tok)
        toks.append(tok)
    return out


def exit_stage_index(tap, L, P):
    per = L // P
    return min(tap // per + 1, P)


def generate_pipeline(P, cfg, heads, num_stages, prompt, threshold, max_new):
    """Pipeline-based inference (`inference.py:406-539`), simulated
    sequentially: stages are FIFO and a token enters stage 1 only after the
    previous token was emitted, so running each message through every stage
    in turn yields the same tokens, exit layers and confidences.  Heads are
    checked only for the decide row; the first firing (or the final) head
    emits.  Returns the same dict shape as `generate_kv_recompute` plus
    exit_stages."""
    if num_stages < 2:
        raise OracleError("config", "pipeline inference needs at least 2 stages")
    prompt = [int(t) for t in prompt]
    if not prompt:
        raise OracleError("config", "prompt must be non-empty")
    if len(prompt) + max_new > cfg.s_max:
        raise OracleError("token", "context exceeds max_seq_len")
    L = cfg.L
    per = L // num_stages
    kv = KV(range(1, L + 1), cfg.s_max, cfg.nh, cfg.h // cfg.nh)
    heads_at = {}
    for hd in heads:
        s = exit_stage_index(hd["tap"], L, num_stages)
        heads_at.setdefault((s, hd["tap"] - (s - 1) * per), []).append(hd)
    conf = {}

    def run_message(x, pos, decide):
        emitted = None
        for s in range(1, num_stages + 1):
            layers = list(range((s - 1) * per + 1, s * per + 1))
            for local in range(0, per + 1):
                if local > 0:
                    x = layer_step(P, layers[local - 1], x, pos, kv, cfg.nh)
                for hd in heads_at.get((s, local), []):
                    r = pos.index(decide)
                    fire, tok, c = exit_decision(head_logits(P, hd, x[r]), threshold)
                    conf.setdefault(decide, {})[hd["key"]] = c
                    if emitted is None and (fire or hd["final"]):
                        emitted = (tok, hd["tap"], s)
        return emitted

    t0 = len(prompt)
    emit = run_message(embed(P, cfg.V, prompt, range(t0)), list(range(t0)), t0 - 1)
    tokens, exits, stages = [], [], []
    position = t0 - 1
    for i in range(max_new):
        tokens.append(emit[0])
        exits.append(emit[1])
        stages.append(emit[2])
        if i == max_new - 1:
            break
        position += 1
        emit = run_message(embed(P, cfg.V, [emit[0]], [position]), [position], position)
    return {"tokens": tokens, "exit_layers": exits, "exit_stages": stages,
            "confidences": [conf.get(t0 - 1 + i, {}) for i in range(len(tokens))]}


# --- training exit head (eepipe/autodiff.py:158-179, 301-323) ---------------


def cross_entropy(logits, targets):
    """mean NLL and probs (`_pykernels.py:64-77`)."""
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    z = e.sum(axis=1, keepdims=True)
    n = logits.shape[0]
    logp = (logits - m) - np.log(z)
    return -logp[np.arange(n), targets].sum() / n, e / z


def exit_head_train(x, w, targets, weight=1.0, norm_w=None):
    """Weighted CE of one exit head and its gradients: logits = [rmsnorm](x) @
    w.T; loss = weight * CE; returns (loss, dx, dw, dnorm).
    Restates `run_head` (`model.py:219-230`) + `cross_entropy`
    (`autodiff.py:301-323`) + `matmul(transpose_b)` backward
    (`autodiff.py:170-177`) + `rmsnorm_bwd` (`_pykernels.py:44-49`)."""
    xs = x
    if norm_w is not None:
        inv = 1.0 / np.sqrt(np.mean(x * x, axis=1) + EPS)
        xs = x * inv[:, None] * norm_w[None, :]
    logits = xs @ w.T
    ce, probs = cross_entropy(logits, targets)
    n = x.shape[0]
    g = probs.copy()
    g[np.arange(n), targets] -= 1.0
    g *= weight / n
    dxs = g @ w
    dw = g.T @ xs
    dnorm = None
    dx = dxs
    if norm_w is not None:
        h = x.shape[1]
        dnorm = np.sum(dxs * x * inv[:, None], axis=0)
        gwx = np.sum(dxs * norm_w[None, :] * x, axis=1)
        dx = dxs * norm_w[None, :] * inv[:, None] - x * (inv ** 3 * gwx / h)[:, None]
    return weight * ce, dx, dw, dnorm


# --- optimizers (eepipe/training.py:24-53) ------------------------------------


def sgd_step(params, grads, scale, lr):
    """`SGD.step` (`training.py:28-30`), float64, in place."""
    for name in sorted(grads):
        params[name] -= lr * scale * grads[name]


def adam_step(params, grads, scale, state, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """`Adam.step` (`training.py:44-53`), float64, in place; ``state`` holds
    t, m, v across calls."""
    state["t"] = state.get("t", 0) + 1
    t = state["t"]
    correction = np.sqrt(1 - beta2 ** t) / (1 - beta1 ** t)
    for name in sorted(grads):
        g = grads[name] * scale
        m = state.setdefault(("m", name), np.zeros_like(g))
        v = state.setdefault(("v", name), np.zeros_like(g))
        m += (1 - beta1) * (g - m)
        v += (1 - beta2) * (g * g - v)
        params[name] -= lr * correction * m / (np.sqrt(v) + eps)


# --- training RMSNorm (eepipe/_pykernels.py:36-49) ----------------------------


def rmsnorm_fwd(x, w, eps=EPS):
    """(y, inv_rms) — `rmsnorm_fwd` (`_pykernels.py:36-41`)."""
    inv = 1.0 / np.sqrt(np.mean(x * x, axis=1) + eps)
    return x * inv[:, None] * w[None, :], inv


def rmsnorm_bwd(x, w, inv_rms, gout):
    """(gx, gw) — `rmsnorm_bwd` (`_pykernels.py:44-49`)."""
    h = x.shape[1]
    gw = np.sum(gout * x * inv_rms[:, None], axis=0)
    gwx = np.sum(gout * w[None, :] * x, axis=1)
    gx = gout * w[None, :] * inv_rms[:, None] - x * (inv_rms ** 3 * gwx / h)[:, None]
    return gx, gw
