"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel
launch count, summed time and share of the total."""
import collections, csv, sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        a = agg.setdefault(r[ki].split("(")[0][:70], [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'launches':>8} {'sum ms':>9} {'share':>6}  kernel"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{a[0]:8d} {a[1] / 1e6:9.3f} {100 * a[1] / tot:5.1f}%  {k}")
    lines.append(f"total {tot / 1e6:.3f} ms (ns units in the csv; cold-cache, serialised by ncu)")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
