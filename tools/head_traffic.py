"""Summarise the ncu launch list of tools/time_train_head.py (C2 shape):
per-kernel time / tensor-pipe % / dram bytes of ONE fused train-head call
(the last one in the list), written to profiles/<tag>_train_head_traffic.json
and a text table."""
import json
import sys

from launches import load


def main():
    path, out_json, out_txt = sys.argv[1:4]
    recs = load(path)
    mine = [r for r in recs if "tc::" in r["name"] or "grad_fixup" in r["name"]
            or "loss_sum" in r["name"]]
    call = mine[-5:]  # K1, fixup, loss_sum, K3, K4 of the last call
    traffic = sum(r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0) for r in call)
    t_us = sum(r["gpu__time_duration.sum"] for r in call) / 1e3
    rows = []
    for r in call:
        rows.append({"kernel": r["name"][:70], "us": r["gpu__time_duration.sum"] / 1e3,
                     "tensor_active_pct": r.get(
                         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                     "dram_read": r.get("dram__bytes_read.sum"),
                     "dram_write": r.get("dram__bytes_write.sum")})
    n, h, V = 4096, 2048, 50304
    json.dump({"what": "ncu launch list (cold, serialised) of one fused train exit head call, "
                       "C2 shape n=4096 h=2048 V=50304 bf16",
               "kernels": rows, "traffic_bytes": traffic, "sum_kernel_us": t_us,
               "tflops_6nhv_on_kernel_sum": 6 * n * h * V / (t_us * 1e-6) / 1e12},
              open(out_json, "w"), indent=1)
    with open(out_txt, "w") as f:
        f.write("fused train exit head, C2 shape (n=4096,h=2048,V=50304), ncu launch list "
                "(cold, serialised)\n")
        for r in rows:
            f.write(f"{r['kernel']:70s} {r['us']:8.1f}us tensor_active%={r['tensor_active_pct'] or 0:5.1f} "
                    f"dram_rd={(r['dram_read'] or 0) / 1e6:8.1f}MB dram_wr={(r['dram_write'] or 0) / 1e6:8.1f}MB\n")
        f.write(f"total {t_us:.1f} us, traffic {traffic / 1e6:.1f} MB\n")


if __name__ == "__main__":
    main()
