"""Copy a measurement run (tools/gpu_measure.sh <tag>) from gpurun_out/ into
profiles/: the bench line, the launch list (+ summary) and the ncu --set full
summary of the wedge kernels with DRAM bytes per count call."""
import json, os, shutil, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402
import launch_summary  # noqa: E402

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(tag, config=2, mode="vertex", orient="high"):
    g = os.path.join(ROOT, "gpurun_out")
    p = os.path.join(ROOT, "profiles")
    shutil.copy(os.path.join(g, f"{tag}_bench.json"), os.path.join(p, f"{tag}_bench_c{config}_{mode}.json"))
    shutil.copy(os.path.join(g, f"{tag}_launches.csv"), os.path.join(p, f"{tag}_launches_c{config}_{mode}.csv"))
    with open(os.path.join(p, f"{tag}_launches_c{config}_{mode}.txt"), "w") as f:
        f.write(launch_summary.summarise(os.path.join(g, f"{tag}_launches.csv")) + "\n")
    res = ncu_summary.load(os.path.join(g, f"{tag}_full.ncu-rep"))
    dram = 0.0
    for r in res:
        b = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = r[key].split()
            b += float(v) * UNITS[u]
        r["dram_bytes"] = b
        dram += b
    out = {"config": config, "mode": mode, "orient": orient, "round": tag,
           "command": "ncu --set full --clock-control none --import-source on -k regex:k_(big|small) -s 3 -c 3 "
                      "python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e",
           "dram_bytes_per_launch": dram,
           "note": "one bf_count call = one launch each of the tier kernels listed; dram bytes summed over them",
           "kernels": res}
    json.dump(out, open(os.path.join(p, f"{tag}_ncu_full_c{config}_{mode}.json"), "w"), indent=1)
    print(f"dram bytes per count call {dram:.4g}")
    for r in res:
        print(r["kernel"][:70], r["gpu__time_duration.sum"], f'{r["dram_bytes"] / 1e6:.1f} MB', r["lts__t_sector_hit_rate.pct"])


if __name__ == "__main__":
    main(sys.argv[1])
