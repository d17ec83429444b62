"""Sum the ncu launch list of ONE full-depth C3 decode pass (tools/prof_decode.py
1 1 <ctx>: 32 layers x 5 kernels, one row) into profiles/<tag>_decode_pass_traffic.json:
dram read + write bytes and kernel time of the 160 layer kernels, next to the
pass's algorithmic bytes (bench.decode_pass_bytes) at the same context.

    python tools/decode_traffic.py gpurun_out/launches_decode_ctx192.csv 192 r2
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import C3, decode_pass_bytes  # noqa: E402


def main():
    path, ctx, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = {}
    for r in rows:
        per.setdefault(r["ID"], {"name": r["Kernel Name"]})[r["Metric Name"]] = (
            float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    ks = [v for _, v in sorted(per.items(), key=lambda kv: int(kv[0]))]
    # the pass = the 160 launches after the engine build / short generation
    layer = [k for k in ks if "k_gemv_tma" in k["name"] or "k_attn" in k["name"]]
    L = C3["num_layers"]
    pass_k = layer[-5 * L:]  # prof_decode.py 1 1 ctx: the last 160 layer kernels

    def b(k, m):
        v, u = k[m]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    def t(k):
        v, u = k["gpu__time_duration.sum"]
        return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[u]
    rd = sum(b(k, "dram__bytes_read.sum") for k in pass_k)
    wr = sum(b(k, "dram__bytes_write.sum") for k in pass_k)
    alg = decode_pass_bytes(C3["hidden_dim"], L, ctx)
    out = {"what": f"ncu launch list (cold cache, serialised) of one full-depth C3 decode pass: "
                   f"{len(pass_k)} launches (32 layers x 5 kernels), 1 row at position {ctx}",
           "source": os.path.basename(path), "launches": len(pass_k),
           "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
           "sum_kernel_us": sum(t(k) for k in pass_k), "ctx": ctx, "algorithmic_bytes": alg,
           "ratio": (rd + wr) / alg}
    with open(os.path.join(ROOT, "profiles", f"{tag}_decode_pass_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
