"""7B pipeline-mode generation with a short prompt (for compute-sanitizer)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model, partition  # noqa: E402

model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=8)]
tr = I.generate_pipeline(partition(model, 2, copy=False), prompt, 0.8, 4)
torch.cuda.synchronize()
print("done", tr.tokens)
