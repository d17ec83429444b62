"""Key counters of an ncu --set full report (raw page) per captured kernel."""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM written"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1/smem throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster x"),
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]  # ncu's raw page: second row = the unit of each column
    idx = {h: i for i, h in enumerate(hdr)}
    with open(out, "w") as f:
        f.write(f"ncu --set full summary of {rep.split('/')[-1]} (clock-control none)\n")
        for r in rows[2:]:
            f.write("\n" + r[idx["Kernel Name"]][:150] + "\n")
            for k, label in WANT:
                if k in idx:
                    unit = units[idx[k]].strip()
                    f.write(f"  {label:28s} {r[idx[k]]} {unit}\n")
            stalls = [(h, r[i]) for h, i in idx.items()
                      if h.startswith("smsp__average_warp_latency_issue_stalled_")
                      or (h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct"))]
            vals = []
            for h, v in stalls:
                try:
                    vals.append((float(v), h))
                except ValueError:
                    pass
            vals.sort(reverse=True)
            for v, h in vals[:5]:
                f.write(f"  stall {h.replace('smsp__warp_issue_stalled_', ''):40s} {v:.1f}\n")


if __name__ == "__main__":
    main()
