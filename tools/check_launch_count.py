"""Cross-check the engine's kernel-launch count (bench `gpu_launches`)
against the CUDA kernels CUPTI records for the same generate call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402


def main():
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = bench.prompt_tokens()
    I.generate_kv_recompute(model, prompt, 0.8, 8, 4)
    eng = next(iter(model.__dict__["_ee_engines"].values()))
    torch.cuda.synchronize()
    before = eng.launches
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        I.generate_kv_recompute(model, prompt, 0.8, 64, 4)
        torch.cuda.synchronize()
    ours = [e for e in prof.events() if e.device_type.name == "CUDA" and
            any(k in e.name for k in ("k_gemv", "k_attn", "k_exit_head", "k_rmsnorm_rows",
                                      "k_embed", "k_row_stats", "k_prefill"))]
    print(f"engine count {eng.launches - before}, CUPTI kernels {len(ours)}")


if __name__ == "__main__":
    main()
