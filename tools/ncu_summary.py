"""Summarise an ncu --set full report (raw page) per kernel: time, DRAM bytes,
L2 hit rate, occupancy, issue activity and the top warp stall reasons."""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct"]


def load(path):
    """path: an .ncu-rep, or the CSV of its raw page (ncu -i rep --page raw --csv)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:80]}
        for key in KEYS:
            if key in d:
                k[key] = d[key] + " " + units[hdr.index(key)]
        stalls = {}
        for i, name in enumerate(hdr):
            if name.startswith("smsp__average_warp_latency_issue_stalled_") and name.endswith(".ratio"):
                try:
                    stalls[name.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")] = float(r[i])
                except ValueError:
                    pass
        if not stalls:
            for i, name in enumerate(hdr):
                if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                    try:
                        stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                    except ValueError:
                        pass
        k["top_stalls"] = sorted(stalls.items(), key=lambda x: -x[1])[:8]
        res.append(k)
    return res


if __name__ == "__main__":
    res = load(sys.argv[1])
    print(json.dumps(res, indent=1))
