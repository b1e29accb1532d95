"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import re
import sys


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")[:100]
        v = float(d["Metric Value"])
        u = d["Metric Unit"]
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(u, 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {len(data)}, total device time {tot / 1e6:.3f} ms"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
