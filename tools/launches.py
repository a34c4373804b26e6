"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main(path):
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")[-48:]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-50s %4d %10.1f us  %5.1f%%" % (k, v[0], v[1], 100 * v[1] / tot))
    for name in ("pair_scan", "commit"):
        xs = [float(d["Metric Value"]) / 1e3 for d in data if name in d["Kernel Name"]]
        print(name, len(xs), [round(x, 1) for x in xs[:90]])


if __name__ == "__main__":
    main(sys.argv[1])
