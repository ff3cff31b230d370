"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: share, count, avg µs per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            if d["Metric Unit"] == "ns":
                v /= 1000.0
            elif d["Metric Unit"] == "ms":
                v *= 1000.0
            agg[d["Kernel Name"][:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{100 * sum(v) / tot:5.1f}%  n={len(v):4d}  avg={sum(v) / len(v):8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
