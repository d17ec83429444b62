"""C3 (7B) decode at long context: prompt 1024, 512 new tokens (positions up
to 1535), thresholds 1.0 / 0.8; checks the pipeline mode agrees bitwise with
KV recompute on the first 64 tokens and reports tokens/s."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402


def main():
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=1024)]
    I.generate_kv_recompute(model, prompt[:64], 0.8, 4)
    for thr in (1.0, 0.8):
        torch.cuda.synchronize()
        t = time.perf_counter()
        tr = I.generate_kv_recompute(model, prompt, thr, 512)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"recompute prompt 1024 + 512 new, thr {thr}: {512 / dt:.1f} tok/s "
              f"(incl. prefill), mean exit {tr.mean_exit_layer:.2f}")
    reco = I.generate_kv_recompute(model, prompt, 0.8, 64)
    pipe = I.generate_pipeline(partition(model, 4, copy=False), prompt, 0.8, 64)
    print("pipeline == recompute (64 tokens, prompt 1024):",
          reco.tokens == pipe.tokens and reco.exit_layers == pipe.exit_layers
          and reco.confidences == pipe.confidences)


if __name__ == "__main__":
    main()
