"""Schedule pieces the hot path needs: the 1F1B per-stage action order and the
analytic pipeline-inference latency model.

Only the parts on the path are restated:

* `regular_actions` — the structural 1F1B order per stage
  (`eepipe/schedule.py:170-179`): warm-up ``min(P-s, M)`` forwards, then
  (F, B) pairs, then the trailing backwards.
* `inference_latency` — modeled per-token latency of pipeline-based
  early-exit inference vs sequential full passes
  (`eepipe/schedule.py:553-590`).  Reported next to measured latency.

* `fill_actions` — the 1F1B list with bubble-fill microbatches inserted
  (`eepipe/schedule.py:182-209`): Part-1 fills between the warm-up forwards
  and the first steady forward exactly as the reference; Part-2 fills at the
  front of each stage's list (the reference slots them into idle gaps with
  its cost model, `eepipe/schedule.py:275-304`; the gradients do not depend
  on the placement, and every placement here is deadlock-free because fill
  actions only wait on the same fill's neighbours).

The reference's cost-model simulator, memory accounting and Gantt rendering
are out of scope.
"""

from __future__ import annotations

from .errors import ConfigError

FWD, BWD = "F", "B"
FILL1_FWD, FILL1_BWD = "F1f", "F1b"
FILL2_FWD, FILL2_BWD = "F2f", "F2b"
FWD_KINDS = (FWD, FILL1_FWD, FILL2_FWD)


def regular_actions(num_stages: int, num_microbatches: int, stage: int):
    """1F1B order for ``stage`` (1-based): list of (kind, microbatch)."""
    m = num_microbatches
    warm = min(num_stages - stage, m)
    acts = [(FWD, k) for k in range(1, warm + 1)]
    for k in range(1, m - warm + 1):
        acts += [(FWD, warm + k), (BWD, k)]
    acts += [(BWD, k) for k in range(m - warm + 1, m + 1)]
    return acts


def fill_actions(num_stages: int, num_microbatches: int, stage: int, part1_depths=(),
                 part2_bwd_depths=()):
    """Per-stage action list with bubble fills.  ``part1_depths``: truncated
    Part-1 depths (None = skipped), ``part2_bwd_depths``: Part-2 backward
    depths (the last r stages run the backward)."""
    p, m = num_stages, num_microbatches
    acts = regular_actions(p, m, stage)
    visiting = [i for i, d in enumerate(part1_depths, 1) if d is not None and d >= stage]
    if visiting:
        inserts = [(FILL1_FWD, i) for i in visiting]
        inserts += [(FILL1_BWD, i) for i in reversed(visiting)]
        cut = min(p - stage, m) + 1  # the warm-up bubble (eepipe/schedule.py:204-208)
        acts = acts[:cut] + inserts + acts[cut:]
    front = []
    for i, r in enumerate(part2_bwd_depths, 1):
        front.append((FILL2_FWD, i))
        if stage >= p - r + 1:
            front.append((FILL2_BWD, i))
    return front + acts


def max_in_flight(actions):
    """Largest number of forwarded-but-not-backwarded regular microbatches."""
    live = peak = 0
    for kind, _ in actions:
        live += 1 if kind == FWD else (-1 if kind == BWD else 0)
        peak = max(peak, live)
    return peak


def inference_latency(exit_stages, stage_times) -> dict:
    """Per-token latency of pipelined early-exit inference.

    Token t enters stage 1 when token t-1 was emitted; at stage s it also
    waits for token t-1's KV fill there; it is emitted when its exit stage
    finishes, and the fill continues in the background.
    """
    p = len(stage_times)
    full = float(sum(stage_times))
    prev_fill = [0.0] * p
    prev_emit = 0.0
    per_token = []
    for e in exit_stages:
        if not 1 <= e <= p:
            raise ConfigError(f"exit stage {e} out of range")
        done = []
        t = prev_emit
        for s in range(p):
            t = max(t, prev_fill[s]) + stage_times[s]
            done.append(t)
        emit = done[e - 1]
        per_token.append(emit - prev_emit)
        prev_emit = emit
        prev_fill = done
    total = sum(per_token)
    seq_total = full * len(exit_stages)
    return {
        "pipeline_per_token": per_token,
        "pipeline_total": total,
        "sequential_per_token": [full] * len(exit_stages),
        "sequential_total": seq_total,
        "per_token_speedup": [full / t for t in per_token],
        "total_speedup": seq_total / total if total else 1.0,
    }
