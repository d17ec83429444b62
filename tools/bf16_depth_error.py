"""How far the bf16 perf path drifts from the float64 oracle with depth, on
the SAME bf16-rounded weights (the 16-layer 7B-width slice of SURVEY B.3):
per-tap relative error of the prompt rows' hidden states (GPU tiled bf16
prefill of 8 rows = the decode GEMV chain vs `ee_oracle.layer_step`), and
the exit_l8 head's confidence on the last row computed from each.  This is
the error budget the end-to-end bf16 parity tolerances are derived from.

    python tools/bf16_depth_error.py > profiles/r2_bf16_depth_error.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import ee_oracle as O  # noqa: E402
from paper_2312_04916_b200 import inference as I  # noqa: E402
from paper_2312_04916_b200.model import ExitSpec, ModelConfig, build_model, model_from_arrays  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    cfg = ModelConfig(L, 4096, 32, 50304, 2048, exits=(ExitSpec(L // 2, "minimalistic", 0.1),))
    t0 = time.time()
    host = build_model(cfg, 0)
    dev = {k: torch.from_numpy(p.data).to("cuda").bfloat16() for k, p in host.params.items()}
    P = {k: v.float().cpu().double().numpy() for k, v in dev.items()}
    del host
    m = model_from_arrays(cfg, dev)
    print(f"# L={L} 7B-width slice, reference init seed 0 rounded to bf16 "
          f"(built in {time.time() - t0:.0f} s)")
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, 50304, size=8)]
    n = len(prompt)
    taps = I.prefill_taps(m, prompt, dtype="bf16")
    taps32 = I.prefill_taps(m, prompt, dtype="fp32")
    kv = O.KV(range(1, L + 1), cfg.max_seq_len, 32, 128)
    x = O.embed(P, 50304, prompt, range(n))
    head = {"kind": "minimalistic", "out": f"exit_l{L // 2}.out"}
    print(" tap  rel_err_bf16   rel_err_fp32path   |x|")
    for l in range(1, L + 1):
        x = O.layer_step(P, l, x, list(range(n)), kv, 32)
        e16 = np.linalg.norm(taps[l] - x) / np.linalg.norm(x)
        e32 = np.linalg.norm(taps32[l] - x) / np.linalg.norm(x)
        print(f"{l:4d}  {e16:.3e}     {e32:.3e}         {np.linalg.norm(x[-1]):.1f}")
        if l == L // 2:
            ref = O.head_logits(P, head, x[-1])
            _, rt, rc = O.exit_decision(ref, 1.0)
            lg, tok, conf, _ = I.head_logits(m, f"exit_l{L // 2}", taps[l][-1:], dtype="bf16")
            lerr = np.linalg.norm(lg[0] - ref) / np.linalg.norm(ref)
            print(f"      exit_l{L // 2} on the last row: reference conf {rc:.5f} (token {rt}), "
                  f"bf16 path conf {conf[0]:.5f} (token {tok[0]}): conf rel dev "
                  f"{abs(conf[0] - rc) / rc:.2e}, logits rel err {lerr:.2e}, "
                  f"logit abs err max {np.abs(lg[0] - ref).max():.3e}")


if __name__ == "__main__":
    main()
