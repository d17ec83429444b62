"""Pipeline vs KV-recompute bitwise check on the 7B model with a 1024-token
prompt (prefill through the tcgen05 GEMM), reporting the first difference."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402


def main():
    n_prompt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=n_prompt)]
    reco = I.generate_kv_recompute(model, prompt, 0.8, 32)
    pipe = I.generate_pipeline(partition(model, P, copy=False), prompt, 0.8, 32)
    print("tokens equal", reco.tokens == pipe.tokens, "exits equal", reco.exit_layers == pipe.exit_layers)
    for i, (a, b) in enumerate(zip(reco.confidences, pipe.confidences)):
        if a != b:
            print("first conf diff at", i, {k: (a.get(k), b.get(k)) for k in set(a) | set(b)})
            break
    else:
        print("confidences equal")


if __name__ == "__main__":
    main()
