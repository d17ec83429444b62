"""Schedule pieces the hot path needs: the 1F1B per-stage action order and the
analytic pipeline-inference latency model.

Only the parts on the path are restated:

* `regular_actions` — the structural 1F1B order per stage
  (`eepipe/schedule.py:170-179`): warm-up ``min(P-s, M)`` forwards, then
  (F, B) pairs, then the trailing backwards.
* `inference_latency` — modeled per-token latency of pipeline-based
  early-exit inference vs sequential full passes
  (`eepipe/schedule.py:553-590`).  Reported next to measured latency.

* `CostModel`, `simulate` (+ `Timeline`, `Event`, `analytic_span`) — the
  discrete-event model the executor takes its per-stage order from
  (`eepipe/schedule.py:41-122`, `124-348`): structural lists with Part-1
  fills between warm-up and steady phase, earliest-start list scheduling
  along the forward / backward chains, then Part-2 fill chains packed into
  the idle gaps (earliest fit), validated.  `Timeline.order(s)` is what a
  stage executes.
* `fill_actions` — a purely structural fill placement (Part-2 at the front
  of each list) kept for callers without a cost model.

Memory accounting (`peak_memory`), replay verification and Gantt rendering
are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

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


# ---------------------------------------------------------------------------
# Discrete-event schedule model (eepipe/schedule.py:41-348)
# ---------------------------------------------------------------------------

VARIANTS = ("standard", "eager-exit", "deferred-exit")


@dataclass(frozen=True)
class CostModel:
    """Abstract per-step costs (`eepipe/schedule.py:41-80`): forward /
    backward time per stage, per-exit forward / backward time, early exits
    per stage (the final head always sits on the last stage and is computed
    eagerly), embedding time on stage 1, point-to-point latency; the
    memory-dimension fields are carried for API compatibility."""

    num_stages: int
    num_microbatches: int
    fwd_time: float = 1.0
    bwd_time: float = 2.0
    exit_fwd_time: float = 0.5
    exit_bwd_time: float = 1.0
    exit_counts: tuple = ()
    seq_len: int = 64
    microbatch_size: int = 4
    vocab_size: int = 256
    hidden_dim: int = 64
    layers_per_stage: int = 2
    embed_fwd_time: float = 0.0
    p2p_latency: float = 0.0

    def __post_init__(self):
        if self.num_stages < 1 or self.num_microbatches < 1:
            raise ConfigError("need at least one stage and one microbatch")
        if min(self.fwd_time, self.bwd_time, self.exit_fwd_time, self.exit_bwd_time) <= 0:
            raise ConfigError("all times must be positive")
        counts = tuple(self.exit_counts) if self.exit_counts else (0,) * self.num_stages
        if len(counts) != self.num_stages:
            raise ConfigError("exit_counts length must equal num_stages")
        object.__setattr__(self, "exit_counts", counts)

    def early_exits_on(self, stage):
        return self.exit_counts[stage - 1]

    def exit_stages(self):
        return [s for s in range(1, self.num_stages + 1) if self.exit_counts[s - 1]]


@dataclass(frozen=True)
class Event:
    kind: str
    mb: int  # regular microbatch (1-based) or fill index
    stage: int
    start: float = 0.0
    end: float = 0.0

    @property
    def duration(self):
        return self.end - self.start

    def tag(self):
        return (self.kind, self.mb)


@dataclass
class Timeline:
    """Simulated iteration (`eepipe/schedule.py:106-121`)."""

    cost: CostModel
    variant: str
    fill_plan: object
    events: list  # per stage, execution order
    span: float
    busy: list
    decomposition: dict
    bubble_assumption_violated: bool
    part1_depths: list = field(default_factory=list)

    def stage_events(self, stage):
        return self.events[stage - 1]

    def order(self, stage):
        return [e.tag() for e in self.events[stage - 1]]


def _duration_fn(cost: CostModel, variant: str):
    """(kind, stage) -> duration (`eepipe/schedule.py:124-167`).  Eager exits
    add their forward to the forward step and their backward to the
    backward step; deferred exits run forward + backward inside the backward
    step; the final head is always forward-eager on the last stage."""
    last = cost.num_stages

    def forward(stage, exits):
        t = cost.fwd_time + (cost.embed_fwd_time if stage == 1 else 0.0)
        if exits and variant == "eager-exit":
            t += cost.exit_fwd_time * cost.early_exits_on(stage)
        return t + (cost.exit_fwd_time if stage == last else 0.0)

    def backward(stage, exits):
        t = cost.bwd_time
        if exits:
            k = cost.early_exits_on(stage)
            if variant == "eager-exit":
                t += cost.exit_bwd_time * k
            elif variant == "deferred-exit":
                t += (cost.exit_fwd_time + cost.exit_bwd_time) * k
        return t + (cost.exit_bwd_time if stage == last else 0.0)

    def duration(kind, stage):
        if kind == FWD:
            return forward(stage, True)
        if kind == BWD:
            return backward(stage, True)
        if kind == FILL1_FWD:  # backbone only: the fill's exits run in its backward
            return cost.fwd_time + (cost.embed_fwd_time if stage == 1 else 0.0)
        if kind == FILL1_BWD:
            return cost.bwd_time + (cost.exit_fwd_time + cost.exit_bwd_time) * \
                cost.early_exits_on(stage)
        if kind == FILL2_FWD:
            return forward(stage, False)
        if kind == FILL2_BWD:
            return backward(stage, variant == "deferred-exit")
        raise ValueError(kind)

    return duration


def build_action_lists(cost: CostModel, variant: str, fill_plan=None):
    """Structural per-stage lists with the Part-1 fills slotted between the
    warm-up forwards and the first steady forward (`eepipe/schedule.py:
    182-209`).  Returns (lists, truncated Part-1 depths)."""
    from .bubblefill import truncated_part1_depths
    p, m = cost.num_stages, cost.num_microbatches
    lists = [regular_actions(p, m, s) for s in range(1, p + 1)]
    depths: list = []
    if fill_plan is not None and not fill_plan.empty:
        if variant == "eager-exit":
            raise ConfigError("bubble filling requires the deferred-exit or standard variant")
        if fill_plan.num_stages != p:
            raise ConfigError("fill plan stage count does not match the cost model")
        if m < p:
            raise ConfigError("bubble filling needs at least P microbatches")
        depths = truncated_part1_depths(fill_plan, cost.exit_stages())
        for s in range(1, p + 1):
            lists[s - 1] = fill_actions(p, m, s, depths, ())
    return lists, depths


def _waits_on(kind, mb, stage, p, part1_depths):
    """The cross-stage event an action depends on (`eepipe/schedule.py:
    212-227`), or None."""
    if kind in (FWD, FILL1_FWD, FILL2_FWD):
        return (kind, mb, stage - 1) if stage > 1 else None
    if kind == BWD:
        return (BWD, mb, stage + 1) if stage < p else (FWD, mb, stage)
    if kind == FILL1_BWD:
        d = part1_depths[mb - 1]
        return (FILL1_BWD, mb, stage + 1) if stage < d else (FILL1_FWD, mb, stage)
    if kind == FILL2_BWD:
        return (FILL2_BWD, mb, stage + 1) if stage < p else (FILL2_FWD, mb, stage)
    raise ValueError(kind)


def _schedule_lists(cost, variant, lists, part1_depths):
    """Earliest start of every action given the per-stage order and each
    action's cross-stage dependency plus the p2p latency (the fixed point
    `eepipe/schedule.py:230-260` computes).  The actions form a DAG (stage
    order edges + one dependency edge each); start times follow from one
    topological pass (Kahn's algorithm) over it.  A cycle means the lists
    cannot be executed."""
    p = cost.num_stages
    dur = _duration_fn(cost, variant)
    index = {(kind, mb, s): (s, i) for s in range(1, p + 1)
             for i, (kind, mb) in enumerate(lists[s - 1])}
    # in-degree: the stage predecessor (i > 0) and the dependency (if any)
    waiting = {}
    children = {}
    for (kind, mb, s), node in index.items():
        dep = _waits_on(kind, mb, s, p, part1_depths)
        n_in = (node[1] > 0) + (dep is not None)
        waiting[node] = n_in
        if dep is not None:
            if dep not in index:
                raise ConfigError("action lists deadlock: unsatisfiable dependency")
            children.setdefault(index[dep], []).append(node)
    start_of, end_of = {}, {}
    dep_ready = {}
    frontier = [node for node, n in waiting.items() if n == 0]
    while frontier:
        s, i = frontier.pop()
        kind, mb = lists[s - 1][i]
        t0 = max(end_of.get((s, i - 1), 0.0), dep_ready.get((s, i), 0.0))
        start_of[(s, i)] = t0
        end_of[(s, i)] = t0 + dur(kind, s)
        released = [(s, i + 1)] if i + 1 < len(lists[s - 1]) else []
        for c in children.get((s, i), ()):
            dep_ready[c] = end_of[(s, i)] + cost.p2p_latency
            released.append(c)
        for c in released:
            waiting[c] -= 1
            if waiting[c] == 0:
                frontier.append(c)
    if len(end_of) != len(index):
        raise ConfigError("action lists deadlock: unsatisfiable dependency")
    events = []
    for s in range(1, p + 1):
        row = []
        for i, (kind, mb) in enumerate(lists[s - 1]):
            row.append(Event(kind, mb, s, start_of[(s, i)], end_of[(s, i)]))
        events.append(row)
    return events


def _idle_gaps(stage_events):
    """Idle intervals [(start, end)] of one stage, the open tail last."""
    ends = [0.0]
    for e in stage_events:
        ends.append(max(ends[-1], e.end))
    gaps = [(busy_until, e.start) for busy_until, e in zip(ends, stage_events)
            if e.start > busy_until]
    return gaps + [(ends[-1], float("inf"))]


def _first_fit(gaps, floor, d):
    """Earliest start >= floor of a d-long slot inside one of the gaps."""
    for g0, g1 in gaps:
        t = max(g0, floor)
        if t + d <= g1 + 1e-9:
            return t
    return max(gaps[-1][0], floor)


def _pack_part2(cost, variant, events, plan):
    """Part-2 chains (forward through every stage, then backward through the
    last r stages) placed into idle time without moving existing events:
    each element at the earliest fitting gap after its chain predecessor
    (+ p2p) and after the previous element of the same kind on that stage
    (the same-kind order is kept; `eepipe/schedule.py:275-304`)."""
    p = cost.num_stages
    dur = _duration_fn(cost, variant)
    kind_floor: dict = {}
    for i, r in enumerate(plan.part2_bwd_depths, 1):
        chain = [(FILL2_FWD, s) for s in range(1, p + 1)] + \
                [(FILL2_BWD, s) for s in range(p, p - r, -1)]
        t_ready = 0.0
        for kind, s in chain:
            d = dur(kind, s)
            t = _first_fit(_idle_gaps(events[s - 1]),
                           max(t_ready, kind_floor.get((kind, s), 0.0)), d)
            events[s - 1].append(Event(kind, i, s, t, t + d))
            events[s - 1].sort(key=lambda e: e.start)
            kind_floor[(kind, s)] = t + d
            t_ready = t + d + cost.p2p_latency
    return events


def _check_timeline(cost, events, part1_depths):
    p = cost.num_stages
    end = {(e.kind, e.mb, e.stage): e.end for evs in events for e in evs}
    start = {(e.kind, e.mb, e.stage): e.start for evs in events for e in evs}
    for evs in events:
        for a, b in zip(evs, evs[1:]):
            if b.start < a.end - 1e-9:
                raise AssertionError(f"overlapping events on stage {a.stage}")
    for key, t0 in start.items():
        dep = _waits_on(key[0], key[1], key[2], p, part1_depths)
        if dep is not None and t0 < end[dep] + cost.p2p_latency - 1e-9:
            raise AssertionError(f"event {key} starts before its dependency {dep}")


def analytic_span(cost: CostModel, variant: str) -> dict:
    """First microbatch's forwards + last stage's steady phase + last
    microbatch's backwards (`eepipe/schedule.py:321-330`)."""
    p, m = cost.num_stages, cost.num_microbatches
    dur = _duration_fn(cost, variant)
    warm = sum(dur(FWD, s) for s in range(1, p + 1))
    steady = (m - 1) * (dur(FWD, p) + dur(BWD, p)) + dur(BWD, p)
    cool = sum(dur(BWD, s) for s in range(1, p))
    return {"warmup": warm, "steady": steady, "cooldown": cool, "total": warm + steady + cool}


def simulate(cost: CostModel, variant: str, fill_plan=None) -> Timeline:
    """The timeline the executor follows (`eepipe/schedule.py:333-348`)."""
    if variant not in VARIANTS:
        raise ConfigError(f"unknown variant {variant!r}")
    if variant == "standard":
        cost = replace(cost, exit_counts=(0,) * cost.num_stages)
    lists, depths = build_action_lists(cost, variant, fill_plan)
    events = _schedule_lists(cost, variant, lists, depths)
    if fill_plan is not None and fill_plan.part2_bwd_depths:
        events = _pack_part2(cost, variant, events, fill_plan)
    _check_timeline(cost, events, depths)
    span = max(e.end for evs in events for e in evs)
    busy = [sum(e.duration for e in evs) for evs in events]
    decomposition = analytic_span(cost, variant)
    violated = fill_plan is None and span > decomposition["total"] + 1e-9
    return Timeline(cost, variant, fill_plan, events, span, busy, decomposition, violated,
                    list(depths))
