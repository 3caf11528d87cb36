"""Per-source-line instruction shares of an ncu source page CSV, sorted by
executed instructions (tools/src_lines.py sorts by stall samples).
usage: python tools/src_inst.py <csv> [top]"""
import collections
import csv
import sys


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


def main(path, top=45):
    rows = list(csv.reader(open(path)))
    per = collections.defaultdict(lambda: [0.0, 0.0, ""])
    fp, hdr, cur = "", None, None
    for r in rows:
        if r and r[0] == "File Path":
            fp = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if not hdr or len(r) <= ie or (r and r[0] == "Function Name"):
            continue
        if r[0]:
            cur = (fp, r[0], r[1])
        if cur is None:
            continue
        e = per[cur[:2]]
        e[0] += num(r[ie]); e[1] += num(r[st]); e[2] = cur[2]
    tot = sum(v[0] for v in per.values()) or 1
    stot = sum(v[1] for v in per.values()) or 1
    acc = 0
    for (f, ln), (i, s_, src) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        acc += i
        print(f"{f[:10]:>10}:{ln:>5} {i / tot * 100:5.1f}% cum {acc / tot * 100:5.1f}% stall {s_ / stot * 100:4.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
