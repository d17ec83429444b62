import time, torch
from torch.profiler import profile, ProfilerActivity
F = torch.nn.functional
B, H, S, D = 2, 16, 2048, 128
q = torch.randn(B, S, H * D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
k = torch.randn(B, S, H * D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
v = torch.randn(B, S, H * D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
split = lambda t: t.view(B, S, H, D).transpose(1, 2)
def it():
    a = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
    a.backward(torch.ones_like(a))
for _ in range(5): it()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    a = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"fwd: cpu {(t1-t0)/20*1e6:.0f} us/call, total {(t2-t0)/20*1e6:.0f} us/call")
g = torch.ones_like(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    a = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
    a.backward(g)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"fwd+bwd: cpu {(t1-t0)/20*1e6:.0f} us/call, total {(t2-t0)/20*1e6:.0f} us/call")
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3): it()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12))
