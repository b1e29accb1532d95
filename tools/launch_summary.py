"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import re
import sys


def summarise(path, top=25, product_only=False):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    harness = [0, 0.0]
    for d in data:
        kn = d["Kernel Name"]
        if product_only and not ("qbgpu" in kn or ("unnamed>" in kn and "at::" not in kn)):
            harness[0] += 1
            v = float(d["Metric Value"]) * {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(
                d["Metric Unit"], 1.0)
            harness[1] += v
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")[:100]
        v = float(d["Metric Value"])
        u = d["Metric Unit"]
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(u, 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {len(data) - harness[0]}, total device time {tot / 1e6:.3f} ms"]
    if product_only:
        out[0] += f" (excluded {harness[0]} harness launches, {harness[1] / 1e6:.3f} ms: torch synthesis, cuBLAS peak probe)"
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    print(summarise(args[0], product_only="--product" in sys.argv))
