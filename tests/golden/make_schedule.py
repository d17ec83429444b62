"""Schedule-simulator golden from the REFERENCE (build container only).

    PYTHONDONTWRITEBYTECODE=1 EEPIPE_BACKEND=python python tests/golden/make_schedule.py

For a sweep of (P, M, exit counts, variant, bubble-fill f/b) runs
`eepipe.schedule.simulate` and records every stage's event order, the span,
the analytic decomposition and the bubble flag in tests/golden/schedule.json.
"""
import json
import os
import sys

os.environ.setdefault("EEPIPE_BACKEND", "python")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from eepipe import schedule as R  # noqa: E402
from eepipe.bubblefill import plan_bubble_fill  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    for P in (2, 3, 4, 8):
        for M in (P, P + 2, 2 * P):
            for ec in [(0,) * P, tuple([1] + [0] * (P - 1)), tuple([0, 1] + [0] * (P - 2)),
                       tuple([1] * P)]:
                for var in ("standard", "eager-exit", "deferred-exit"):
                    for fb in (None, 0.5, 0.25):
                        if fb is not None and (var == "eager-exit" or M < P):
                            continue
                        yield P, M, ec, var, fb


def main():
    out = []
    for P, M, ec, var, fb in cases():
        c = R.CostModel(P, M, exit_counts=ec, embed_fwd_time=0.3, p2p_latency=0.05)
        t = R.simulate(c, var, plan_bubble_fill(P, fb) if fb else None)
        out.append({"P": P, "M": M, "exit_counts": list(ec), "variant": var, "f_over_b": fb,
                     "orders": [[list(a) for a in t.order(s)] for s in range(1, P + 1)],
                     "span": t.span, "decomposition": t.decomposition,
                     "violated": t.bubble_assumption_violated})
    with open(os.path.join(HERE, "schedule.json"), "w") as f:
        json.dump(out, f)
    print("wrote", len(out), "timelines")


if __name__ == "__main__":
    main()
