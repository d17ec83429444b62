"""Time the C3 prefill pass (64 prompt rows through all 32 layers + heads)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402


def main():
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = bench.prompt_tokens()
    for _ in range(2):
        I.generate_kv_recompute(model, prompt, 1.0, 1, 4)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        I.generate_kv_recompute(model, prompt, 1.0, 1, 4)  # prefill only (decides token 1)
    b.record()
    torch.cuda.synchronize()
    print(f"prefill of {len(prompt)} rows: {a.elapsed_time(b) / 5:.2f} ms")


if __name__ == "__main__":
    main()
