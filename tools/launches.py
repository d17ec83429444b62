"""Summarise an ncu --csv launch list: per-kernel-name time share over the
last full-depth decode pass (or all launches)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = int(d["ID"])
            rec = recs.setdefault(key, {"name": d["Kernel Name"], "grid": d["Grid Size"],
                                        "block": d["Block Size"]})
            rec[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [recs[k] for k in sorted(recs)]


def main():
    recs = load(sys.argv[1])
    start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    n = int(sys.argv[3]) if len(sys.argv) > 3 else len(recs)
    sel = recs[start:start + n] if start >= 0 else recs[start:][:n]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in sel:
        a = agg[r["name"][:70]]
        a[0] += 1
        a[1] += r.get("gpu__time_duration.sum", 0.0)
        a[2] += r.get("dram__bytes_read.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'n':>4} {'total_us':>10} {'share':>6} {'avg_us':>8} {'GB/s':>8}  kernel")
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = b / t if t else 0  # bytes/ns = GB/s
        print(f"{c:4d} {t / 1e3:10.1f} {t / tot * 100:5.1f}% {t / c / 1e3:8.2f} {gbs:8.0f}  {k}")
    print(f"total {tot / 1e3:.1f} us over {len(sel)} launches")


if __name__ == "__main__":
    main()
