"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source
line: executed warp instructions and stall samples per line (all inlined copies)."""
import csv, collections, sys


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if len(r) > 8 and r[0] == "Line No"][0]
    h = rows[hi]
    ie = h.index("Instructions Executed")
    st = h.index("Warp Stall Sampling (All Samples)")
    per = collections.defaultdict(lambda: [0.0, 0.0, ""])
    cur_line, cur_src = None, ""
    seen = set()
    for r in rows[hi + 1:]:
        if len(r) <= ie:
            continue
        if r[0]:
            cur_line, cur_src = r[0], r[1]
        if r[2] in seen:
            continue
        seen.add(r[2])
        e = per[cur_line]
        e[0] += num(r[ie])
        e[1] += num(r[st])
        e[2] = cur_src
    tot = sum(v[0] for v in per.values())
    stot = sum(v[1] for v in per.values())
    print(f"total inst {tot:.4g} stall samples {stot:.4g}")
    for ln, (i, s_, src) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:>5} {i / tot * 100:5.1f}% inst {s_ / stot * 100:5.1f}% stall  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
