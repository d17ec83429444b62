"""Top SASS instructions by warp-stall samples of one kernel in an ncu report
(--set full --import-source on), with the stall columns that dominate.

    python tools/ncu_hot.py REPORT.ncu-rep [kernel-regex] [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kre:
        cmd += ["-k", "regex:" + kre]
    cmd += ["--launch-count", "1"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = None
    data = []
    for r in rows:
        if "Address" in r and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(d.get(key, 0) or 0) for d in data)
    data.sort(key=lambda d: -float(d.get(key, 0) or 0))
    print(f"total samples {tot:.0f}")
    for d in data[:top]:
        s = float(d.get(key, 0) or 0)
        print(f"{100 * s / max(tot, 1):5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()
