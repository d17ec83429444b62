"""Time one C2 training step (EE-GPT 1.3B: L=24, h=2048, 16 heads, V=50304,
seq 2048, tied exits at layers 6 (w 0.25) and 12 (w 0.5); microbatch 2,
M microbatches; 1F1B executor at P=1, fused tcgen05 exit heads, fused Adam
on float32 master weights) with CUDA events."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, partition  # noqa: E402
from paper_2312_04916_b200.pipeline import IterationOptions, run_iteration_1f1b  # noqa: E402
from paper_2312_04916_b200.training import Adam, apply_update  # noqa: E402


def c2_config():
    return ModelConfig(24, 2048, 16, 50304, 2048,
                       exits=(ExitSpec(6, "minimalistic", 0.25), ExitSpec(12, "minimalistic", 0.5)),
                       tie_embeddings=True)


def train_step_bench(M=8, mb=2, seq=2048, steps=3, warmup=int(os.environ.get("TS_WARMUP", "4")), stages=1):
    cfg = c2_config()
    master = build_model(cfg, 0, init="device", dtype=torch.float32)
    opt = Adam(3e-4)
    rng = np.random.default_rng(0)
    batches = [rng.integers(0, cfg.vocab_size, size=(M * mb, seq + 1)) for _ in range(steps + warmup)]

    part = partition(master, stages, copy=False)
    computes = []

    def step(i):
        grads, rep = run_iteration_1f1b(part, batches[i], IterationOptions(microbatch_size=mb),
                                        model=master, master_dtype=torch.float32,
                                        stage_computes=computes)
        apply_update(opt, master, grads, computes, 1.0 / M)
        return rep

    import time
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    per = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        t0 = time.perf_counter()
        rep = step(warmup + i)
        torch.cuda.synchronize()
        per.append((time.perf_counter() - t0) * 1e3)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    print("per-step wall ms:", [round(x, 1) for x in per], file=sys.stderr)
    tokens = M * mb * seq
    return {"workload": f"C2 EE-GPT 1.3B training step (L=24, h=2048, V=50304, seq {seq}, "
                        f"microbatch {mb} x {M}, tied exits 6/12, P={stages}, Adam fp32 master)",
            "ms_per_step": ms, "tokens_per_s": tokens / (ms / 1e3), "tokens_per_step": tokens,
            "losses": rep.per_exit_losses,
            "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}


if __name__ == "__main__":
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    mb = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    print(train_step_bench(M=M, mb=mb))
