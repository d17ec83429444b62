import sys, time
sys.argv=["x"]; sys.path.insert(0,".")
import torch, bench
from paper_2312_04916_b200 import inference as I
from paper_2312_04916_b200.model import build_model
print("fresh", bench.bench_train_step(0)["ms_per_step"], flush=True)
print("again", bench.bench_train_step(0)["ms_per_step"], flush=True)
bench.bench_train_head(0, 6000)
print("after head", bench.bench_train_step(0)["ms_per_step"], flush=True)
model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
print("after 7B alloc", bench.bench_train_step(0)["ms_per_step"], flush=True)
I.generate_kv_recompute(model, bench.prompt_tokens(), 0.8, 64, 4)
print("after decode", bench.bench_train_step(0)["ms_per_step"], flush=True)
