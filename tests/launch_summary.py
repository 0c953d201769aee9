"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3,
         "us": 1.0, "ms": 1e3, "s": 1e6}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("dg::<unnamed>::", "").replace("dg::", "")
        us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:48]:48s} {n:8d} {us / 1e3:10.3f} {us / n:10.1f} {100 * us / tot:6.2f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
