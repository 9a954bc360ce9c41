"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
launch count, mean and total duration per kernel name, in first-launch order."""
import csv
import sys
from collections import OrderedDict


def main(path, title=""):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0][:48]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    if title:
        print(title)
    for name, (n, t) in agg.items():
        print(f"{name:48s} n={n:5d} mean={t / n:10.2f} us  total={t / 1e3:9.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
