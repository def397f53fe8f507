"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total/mean device time and share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("vms::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot:.1f} us total")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.1f} us {v[0]:4d}x {v[1] / v[0]:9.1f} us/launch {100 * v[1] / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
