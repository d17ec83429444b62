"""Stress for nondeterminism on the small model, in the shape of
tests/test_gpu_parity.py::test_gpu_modes_bitwise_equal: one model (engines
reused across calls), thresholds x max_deferred, repeated; pipeline and
recompute must agree bitwise every time.  python tools/stress_modes.py [reps]"""
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import gold, small_config  # noqa: E402

from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402

prompt = gold()["small_prompts"][0]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
small = build_model(small_config(), 7)
bad = 0
for rep in range(reps):
    for dtype in ("fp32", "bf16"):
        part = partition(small, 4)
        for thr in (1.0, 6.0 / 64, 0.99 / 64, 0.015775):
            for md in (1, 2, 4):
                p = I.generate_pipeline(part, prompt, thr, 12, dtype=dtype)
                r = I.generate_kv_recompute(small, prompt, thr, 12, md, dtype=dtype)
                if (p.tokens, p.exit_layers, p.confidences) != (r.tokens, r.exit_layers,
                                                                 r.confidences):
                    bad += 1
                    print("MISMATCH rep", rep, dtype, thr, md, flush=True)
                    print("  pipe", p.tokens, p.exit_layers, flush=True)
                    print("  reco", r.tokens, r.exit_layers, flush=True)
                    for i, (a, b) in enumerate(zip(p.confidences, r.confidences)):
                        if a != b:
                            print("  conf", i, a, b, flush=True)
print("mismatches", bad)
