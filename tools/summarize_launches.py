"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total and mean device time, share of the total."""
import csv
import collections
import sys


def main(path, skip_prefix=None):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rdr = csv.DictReader(lines)
    for r in rdr:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
        rows.append((r["Kernel Name"], v))
    agg = collections.OrderedDict()
    for name, us in rows:
        short = name.split("(")[0][:70]
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{len(rows)} launches, {tot:.1f} us total")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{us:10.1f} us {100 * us / tot:5.1f}%  n={n:4d}  mean={us / n:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
