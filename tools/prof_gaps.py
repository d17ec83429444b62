"""GPU idle-gap census of C3 decode (torch.profiler / CUPTI kernel records):
per generated token, the GPU busy time vs wall time, and the histogram of
idle gaps between consecutive kernels (host synchronisation bubbles)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402


def main():
    thr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.8
    ntok = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = bench.prompt_tokens()
    I.generate_kv_recompute(model, prompt, thr, 16, 4)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tr = I.generate_kv_recompute(model, prompt, thr, ntok, 4)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    gaps = []
    pairs = {}
    end = ev[0].time_range.end
    prev = ev[0]
    for e in ev[1:]:
        g = e.time_range.start - end
        if g > 0:
            gaps.append(g)
            if g > 5:
                k = (prev.name[:40], e.name[:40])
                pairs.setdefault(k, [0, 0.0])
                pairs[k][0] += 1
                pairs[k][1] += g
        if e.time_range.end >= end:
            end = e.time_range.end
            prev = e
    gaps.sort()
    big = [g for g in gaps if g > 5]
    print(f"thr={thr} tokens={len(tr.tokens)} kernels={len(ev)} span={span/1e3:.2f} ms "
          f"busy={busy/1e3:.2f} ms idle={(span-busy)/1e3:.2f} ms "
          f"per token: span {span/len(tr.tokens):.0f} us busy {busy/len(tr.tokens):.0f} us")
    print(f"gaps>5us: n={len(big)} sum={sum(big)/1e3:.2f} ms  median={big[len(big)//2] if big else 0:.1f} us "
          f"p90={big[int(len(big)*0.9)] if big else 0:.1f} us max={big[-1] if big else 0:.1f}")
    for (a, b), (c, t) in sorted(pairs.items(), key=lambda x: -x[1][1])[:8]:
        print(f"  gap {c:5d}x {t/1e3:7.2f} ms  after {a!r} before {b!r}")
    print(f"mean exit layer {tr.mean_exit_layer:.2f}, early {sum(1 for e in tr.exit_layers if e < 32)}")
    names = {}
    for e in ev:
        n = e.name[:60]
        names.setdefault(n, [0, 0.0])
        names[n][0] += 1
        names[n][1] += e.time_range.end - e.time_range.start
    for n, (c, t) in sorted(names.items(), key=lambda x: -x[1][1])[:10]:
        print(f"  {c:6d} {t/1e3:8.2f} ms  {n}")


if __name__ == "__main__":
    main()
