"""Per-instruction hot spots of an ncu source page (--print-source sass --csv):
executed instructions and stall samples, grouped into basic-block-like runs."""
import csv, sys, collections


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
    h = rows[hi]
    R = [r for r in rows[hi + 1:] if len(r) > 10]
    ie, st, at = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
    # the page can list the function twice; keep the first copy
    seen = set()
    uniq = []
    for r in R:
        if r[0] in seen:
            break
        seen.add(r[0])
        uniq.append(r)
    tot = sum(num(r[ie]) for r in uniq)
    stot = sum(num(r[st]) for r in uniq)
    print(f"instructions {tot:.4g}  stall samples {stot:.4g}  ({len(uniq)} sass lines)")
    # group consecutive instructions with the same exec count into blocks
    blocks = []
    cur = None
    for i, r in enumerate(uniq):
        c = num(r[ie])
        if cur and cur["count"] == c:
            cur["n"] += 1
            cur["stall"] += num(r[st])
            cur["ops"].append(r[1].strip().split()[0] if not r[1].strip().startswith("@") else r[1].strip().split()[1])
        else:
            cur = dict(start=i, count=c, n=1, stall=num(r[st]), thr=num(r[at]),
                       ops=[r[1].strip().split()[0] if not r[1].strip().startswith("@") else r[1].strip().split()[1]])
            blocks.append(cur)
    blocks.sort(key=lambda b: -b["count"] * b["n"])
    for b in blocks[:top]:
        print(f"{b['start']:5d} n={b['n']:3d} exec={b['count']:.3g} tot={b['count']*b['n']/tot*100:5.1f}% "
              f"stall={b['stall']/stot*100:5.1f}% thr={b['thr']:4.1f} {' '.join(b['ops'][:14])}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
