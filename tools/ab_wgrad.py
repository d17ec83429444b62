import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
import paper_2312_04916_b200.training as T
import time_train_step as S
orig = T._matmul
def plain(params, name, x):
    return x @ params[name]
for rep in range(2):
    for tag, fn in (("fused", orig), ("cublas", plain)):
        T._matmul = fn
        r = S.train_step_bench(M=8, steps=5, warmup=2)
        print(tag, round(r["ms_per_step"], 1), file=sys.stderr)
