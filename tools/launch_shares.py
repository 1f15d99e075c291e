"""Kernel shares of GPU time from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict


def main(path, header=""):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            if d.get("Metric Unit") == "usecond":
                v *= 1e3
            elif d.get("Metric Unit") == "msecond":
                v *= 1e6
            k = d["Kernel Name"][:60]
            tot[k] += v
            cnt[k] += 1
    s = sum(tot.values()) or 1.0
    if header:
        print(header)
    print("# kernel | launches | total ns | share")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k} | {cnt[k]} | {int(v)} | {100 * v / s:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
