"""GPU busy vs idle over one C3 generation (threshold 0.8): torch.profiler
(CUPTI) kernel intervals, merged, against the wall span; per-kernel totals."""
import collections
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
    thr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.8
    new = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = bench.prompt_tokens()
    for _ in range(2):
        I.generate_kv_recompute(model, prompt, thr, new, bench.MAX_DEFERRED)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tr = I.generate_kv_recompute(model, prompt, thr, new, bench.MAX_DEFERRED)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
    span = iv[-1][1] - iv[0][0]
    busy, cur_s, cur_e = 0, iv[0][0], iv[0][1]
    gaps = []
    for s, e in iv[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append(s - cur_e)
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    gaps.sort(reverse=True)
    print(f"threshold {thr}: {len(tr.tokens)} tokens, span {span / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms "
          f"({100 * busy / span:.1f}%), idle {100 - 100 * busy / span:.1f}%, "
          f"{len(gaps)} gaps, largest {[round(g, 1) for g in gaps[:8]]} us")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        a = agg[e.name[:80]]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
        print(f"{t / 1e3:8.2f} ms {c:6d}  {k}")


if __name__ == "__main__":
    main()
