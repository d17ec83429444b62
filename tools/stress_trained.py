"""Nondeterminism hunt on the reference-trained tiny model (bf16): repeats
tests/test_gpu_trained.py::test_trained_bf16_modes_bitwise_equal and reports
which mode deviates from its own first run."""
import json
import os
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
from helpers import GOLD_DIR  # noqa: E402

from paper_2312_04916_b200 import checkpoint as C  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import partition  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
trained = C.load_model(os.path.join(GOLD_DIR, "trained_tiny.ckpt"))
with open(os.path.join(GOLD_DIR, "trained.json")) as f:
    g = json.load(f)
part = partition(trained, 2)
first = {}
stats = {"pipe": 0, "reco": 0, "modes": 0}
for rep in range(reps):
    for pi, prompt in enumerate(g["prompts"]):
        for thr in (0.9, 0.8, 0.5):
            pipe = I.generate_pipeline(part, prompt, thr, 24, dtype="bf16")
            reco = I.generate_kv_recompute(trained, prompt, thr, 24, 4, dtype="bf16")
            kp = (pipe.tokens, pipe.exit_layers, pipe.confidences)
            kr = (reco.tokens, reco.exit_layers, reco.confidences)
            key = (pi, thr)
            if key not in first:
                first[key] = (kp, kr)
            for name, cur, ref in (("pipe", kp, first[key][0]), ("reco", kr, first[key][1])):
                if cur != ref:
                    stats[name] += 1
                    idx = next(i for i, (a, b) in enumerate(zip(cur[2], ref[2])) if a != b)
                    print(f"{name} deviates rep {rep} prompt {pi} thr {thr} at token {idx}:",
                          cur[0][idx] if idx < len(cur[0]) else None, ref[0][idx] if idx < len(ref[0]) else None,
                          cur[2][idx], ref[2][idx], flush=True)
            if kp != kr:
                stats["modes"] += 1
print(stats, "cases", reps * len(g["prompts"]) * 3)
