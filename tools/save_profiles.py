"""Copy a measurement run from gpurun_out/ into profiles/: the bench line, the
launch list (+ per-kernel summary) and the ncu --set full summary of the wedge
kernels of one count call, with the per-count DRAM bytes, kernel time, L2 hit
rate, issue activity, warp instructions per wedge and the SHA-256 of the CUDA
sources the capture measured (bench.py reports the summary as this build's
`roofline.traffic` only when that hash matches).

  python tools/save_profiles.py <tag> <config> <mode> [--bench <json>] [--launches <csv>] [--ncu <rep>]
"""
import argparse
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, ROOT)
import launch_summary  # noqa: E402
import ncu_summary  # noqa: E402

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TUNITS = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3}


def qty(s, table):
    v, u = s.split()
    return float(v) * table.get(u, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("config", type=int)
    ap.add_argument("mode")
    ap.add_argument("--bench")
    ap.add_argument("--launches")
    ap.add_argument("--ncu")
    ap.add_argument("--W", type=float, default=None)
    ap.add_argument("--orient", default="high")
    a = ap.parse_args()
    p = os.path.join(ROOT, "profiles")
    base = f"{a.tag}_c{a.config}_{a.mode}"
    W = a.W
    if a.bench:
        shutil.copy(a.bench, os.path.join(p, f"{base}_bench.json"))
        try:
            W = W or json.loads(open(a.bench).readline())["config"]["W"]
        except Exception:
            pass
    if a.launches:
        shutil.copy(a.launches, os.path.join(p, f"{base}_launches.csv"))
        with open(os.path.join(p, f"{base}_launches.txt"), "w") as f:
            f.write(launch_summary.summarise(a.launches) + "\n")
    if a.ncu:
        import bench  # the same source hash bench.py computes
        res = ncu_summary.load(a.ncu)
        dram = t_ms = inst = 0.0
        issue, l2 = [], []
        import math
        missing = []
        for r in res:
            t = qty(r["gpu__time_duration.sum"], TUNITS)
            t_ms += t
            b = sum(qty(r[k], UNITS) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            if math.isnan(b):  # ncu returned no value for this launch's counters
                missing.append(r["kernel"][:60])
                r["dram_bytes"] = None
                continue
            r["dram_bytes"] = b
            dram += b
            inst += float(r["smsp__inst_executed.sum"].split()[0])
            issue.append((t, float(r["smsp__issue_active.avg.pct_of_peak_sustained_active"].split()[0])))
            l2.append((b, float(r["lts__t_sector_hit_rate.pct"].split()[0])))
        wsum = lambda xs: sum(w * v for w, v in xs) / max(sum(w for w, _ in xs), 1e-30)
        out = {"config": a.config, "mode": a.mode, "orient": a.orient, "round": a.tag,
               "src_sha": bench.src_sha(),
               "command": "tools/ncu_kernel.sh: ncu --set full --clock-control none --import-source on "
                          "-k regex:<wedge kernels> (one count call) python bench.py --steps 1 --warmup 1",
               "dram_bytes_per_launch": dram, "kernel_ms": t_ms,
               "l2_hit_pct": wsum(l2), "issue_active_pct": wsum(issue),
               "warp_inst_per_wedge": (inst / W if W else None) if not missing else None,
               "limiter": "L1/shared-memory wavefronts, shared-atomic latency and issue (see per-kernel stalls); "
                          "DRAM is not the binding unit",
               "note": "one bf_count call = one launch each of the kernels listed; bytes, time and instructions "
                       "summed over them (ncu serialises and flushes caches: shares matter, not absolutes)",
               "counters_missing_for": missing,
               "kernels": res}
        json.dump(out, open(os.path.join(p, f"{base}_ncu_full.json"), "w"), indent=1)
        print(f"{base}: dram {dram / 1e9:.3f} GB, kernels {t_ms:.3f} ms, L2 hit {wsum(l2):.1f}%, "
              f"issue {wsum(issue):.1f}%, warp-inst/wedge {out['warp_inst_per_wedge']}")


if __name__ == "__main__":
    main()
