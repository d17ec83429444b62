"""Localise run-to-run nondeterminism at long prompts: (1) repeated prefill
taps, (2) repeated short recompute generations, (3) repeated standalone
attention calls on a reused workspace."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_04916_b200 import _lib, inference as I  # noqa: E402
from paper_2312_04916_b200._lib import call, ptr, stream_ptr  # noqa: E402
from paper_2312_04916_b200.model import build_model  # noqa: E402


def attn_repeat():
    lib = _lib.load()
    nh, dh, smax = 32, 128, 2048
    h = nh * dh
    g = torch.Generator(device="cuda").manual_seed(0)
    kc = torch.randn((smax, h), generator=g, device="cuda").bfloat16()
    vc = torch.randn((smax, h), generator=g, device="cuda").bfloat16()
    for pos in ([260], [256, 257, 258, 259, 260], list(range(260)), [1000], list(range(1000, 1005))):
        m = len(pos)
        q = torch.randn((m, h), generator=g, device="cuda") * 0.3
        pd = torch.tensor(pos, dtype=torch.int32, device="cuda")
        ws = torch.zeros(lib.ee_workspace_bytes(_lib.EE_OP_ATTENTION, m, h, 0, nh, smax),
                         dtype=torch.uint8, device="cuda")
        outs = []
        for _ in range(50):
            out = torch.empty((m, h), dtype=torch.bfloat16, device="cuda")
            call("ee_decode_attention", ptr(q), m, ptr(pd), int(max(pos)), ptr(kc), ptr(vc), nh,
                 dh, _lib.EE_BF16, ptr(out), ptr(ws), ws.numel(), stream_ptr())
            outs.append(out)
        torch.cuda.synchronize()
        bad = sum(not torch.equal(o, outs[0]) for o in outs)
        print("attn m=%d pos[-1]=%d: %d/50 differ" % (m, pos[-1], bad), flush=True)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 260
    reco_only = len(sys.argv) > 2
    if not reco_only:
        attn_repeat()
    model = build_model(bench.c3_config(), 0, init="device", dtype=torch.bfloat16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 50304, size=n)]
    first = []
    if not reco_only:
        a = I.prefill_taps(model, prompt)
        b = I.prefill_taps(model, prompt)
        first = [l for l in range(len(a)) if not np.array_equal(a[l], b[l])]
        print("prefill taps differ at layers:", first[:5], flush=True)
    if first:
        l = first[0]
        rows = np.nonzero((a[l] != b[l]).any(axis=1))[0]
        print("  rows differing at layer", l, rows[:20], len(rows))
    r = [I.generate_kv_recompute(model, prompt, 0.8, 3) for _ in range(4)]
    for x in r:
        print("reco", x.tokens, x.exit_layers, x.confidences[1].get("exit_l8"))


if __name__ == "__main__":
    main()
