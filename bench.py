#!/usr/bin/env python
"""bench.py -- exact butterfly counting throughput on B200 (one JSON line).

Workload (default): BASELINE.json configs[1] = config 2, Chung-Lu 1M x 200K,
10M edges, gamma 2.1/2.1, seed 2, exact per-vertex counts, exact-degree ranking.

A "step" is one pass of the whole hot path over the graph:
bf_graph_create (ingest, validate, dedup check, degrees) -> bf_rank (ranking,
ranked CSR, wedge prefix, plan) -> bf_count_vertex (wedge kernels, finalize,
centre pass, un-rename, allreduce for N > 1) -> bf_graph_destroy, with the edge
list already resident in HBM.  value = W / t_step (wedges/s) where W is the
number of wedges the method processes under the ranking (reading Z10).

  python bench.py [--gpus N --steps K --warmup W] [--config k] [--mode vertex|edge|total]
  python bench.py --impl reference ...   # the CPU oracle on a bounded sample

For N > 1 it is launched by torch.distributed.run, one rank per GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "wedges/sec and edges/sec, exact per-vertex count, 1/2/4/8 B200; % HBM roofline"
UNIT = "wedges/s"
CONFIG_DESC = {
    1: "c1: uniform 2,000 x 1,500, 20,000 distinct edges, seed 1",
    2: "c2: Chung-Lu |U|=1M, |V|=200K, 10M distinct edges, gamma 2.1/2.1, seed 2",
    3: "c3: Chung-Lu 3M x 3M, 100M distinct edges, gamma 2.0/2.5, planted K_{200,300}, seed 3",
    4: "c4: 20M users (Geometric mean 7) x 30K items (Zipf 1.2), seed 4",
    5: "c5: Chung-Lu 8M x 3M, 300M distinct edges, gamma 1.9/1.9, seed 5",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--mode", choices=["vertex", "edge", "total"], default="vertex")
    p.add_argument("--rank", default=None, help="ranking (default: the config's)")
    p.add_argument("--orient", default="auto", choices=["auto", "low", "high"])
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target wall time of the CPU-oracle sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []  # (host arrival time, csv line)
        self.windows = []  # timed regions (host time)

    def _nvml_open(self):
        """In-process NVML (what nvidia-smi itself reads): a looping nvidia-smi process beside the
        benchmark stalls the launching thread for milliseconds whenever one of its queries lands
        inside a step (r02c/r02f: +1.2 to +2.0 ms per c2 step with a second sample in the region),
        so the same clocks and event reasons are read here from a thread.  BF_CLOCKS=smi selects
        the nvidia-smi loop."""
        import pynvml
        pynvml.nvmlInit()
        idx = self.idx
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        if vis:
            ent = [x.strip() for x in vis.split(",") if x.strip()]
            if idx < len(ent) and ent[idx].isdigit():
                idx = int(ent[idx])
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        return pynvml, h, smax

    def _nvml_loop(self, pynvml, h, smax):
        bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        while not self.stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                f = [str(self.idx), str(sm), str(smax), "", hex(r)] + ["Active" if r & b else "Not Active" for b in bits]
                self.lines.append((time.time(), ", ".join(f)))
            except Exception:
                pass
            self.stop.wait(0.05)

    def __enter__(self):
        self.stop = threading.Event()
        self.source = "nvidia-smi"
        if os.environ.get("BF_CLOCKS", "nvml") != "smi":
            try:
                args = self._nvml_open()
                self.t = threading.Thread(target=self._nvml_loop, args=args, daemon=True)
                self.t.start()
                self.source = "nvml"
                return self
            except Exception:
                pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def timed(self, t0: float, t1: float):
        self.windows.append((t0, t1))

    def wait_first(self, limit: float = 5.0):
        t = time.time()
        while (self.proc or self.source == "nvml") and not self.lines and time.time() - t < limit:
            time.sleep(0.02)

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Samples that arrived during a timed region (plus the sampling period,
        as a sample reports the interval before it); if a region was shorter
        than the period, the first sample after each region."""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for t, ln in self.lines if any(a <= t <= b + 0.06 for a, b in self.windows)]
        if not inside:
            for a, b in self.windows:
                after = [ln for t, ln in self.lines if t >= a]
                inside += after[:1]
        for ln in inside:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "period_ms": 50, "source": self.source}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(g, W: int, target_s: float, mode: str):
    """Time the plain CPU oracle (as it stands) on a bounded sample of the
    workload: the first K vertices of its enumeration side (ids are a random
    permutation, so a prefix is a uniform sample), split over the host cores
    as independent single-threaded shards.  Returns the extrapolated full-graph
    rate in wedges/s (W / estimated full oracle time)."""
    import multiprocessing as mp

    import oracle
    og = oracle.OracleGraph(g.n_u, g.n_v, g.edges)
    X = og.cheap_side()
    deg_y = np.bincount(g.edges[:, 1 - X], minlength=(g.n_u, g.n_v)[1 - X]).astype(np.int64)
    cost = np.zeros((g.n_u, g.n_v)[X], np.int64)
    np.add.at(cost, g.edges[:, X].astype(np.int64), deg_y[g.edges[:, 1 - X]])
    cost = cost * 2 + 1  # two walks per x (pass over N2(x), then the per-edge/centre walk)
    total_cost = int(cost.sum())
    P = max(1, len(os.sched_getaffinity(0)))
    vert, edge = mode == "vertex", mode == "edge"
    # calibrate single-thread speed on a short prefix
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 0.3 and k < len(cost):
        hi = min(len(cost), k + 64)
        og.count_range(X, k, hi, vertex=vert, edge=edge)
        k = hi
    rate = cost[:k].sum() / max(time.perf_counter() - t0, 1e-6)
    budget = rate * target_s * P
    csum = np.cumsum(cost)
    K = int(np.searchsorted(csum, budget)) + 1
    K = max(P, min(K, len(cost)))
    cuts = np.searchsorted(csum[:K], np.linspace(0, csum[K - 1], P + 1)[1:-1]).tolist()
    bounds = list(zip([0] + cuts, cuts + [K]))
    ctx = mp.get_context("fork")
    global _OG, _ARGS
    _OG, _ARGS = og, (X, vert, edge)
    t0 = time.perf_counter()
    with ctx.Pool(P) as pool:
        cpu = pool.map(_oracle_shard, bounds)
    wall = time.perf_counter() - t0
    sample_cost = int(csum[K - 1])
    est_full = wall * total_cost / sample_cost
    og.close()
    return dict(value=W / est_full, unit=UNIT, cores=P, kind="oracle",
                sample=(f"first {K} of {len(cost)} side-{'UV'[X]} vertices ({100.0 * sample_cost / total_cost:.3f}% "
                        f"of the oracle's 2*sum(deg^2) steps), {P} single-threaded shards, {wall:.2f} s wall, "
                        f"{sum(cpu):.2f} s CPU; full run extrapolated to {est_full:.1f} s"),
                est_full_s=est_full, sample_wall_s=wall)


_OG = None
_ARGS = None


def _oracle_shard(b):
    lo, hi = b
    X, vert, edge = _ARGS
    t = time.process_time()
    _OG.count_range(X, lo, hi, vertex=vert, edge=edge)
    return time.process_time() - t


def algorithmic_bytes(mode: str, W: int, m: int, n: int, P: int) -> int:
    """SURVEY 8(d) per-unit bytes: W wedges, m forward
    slots, P distinct endpoint pairs, n vertices."""
    if mode == "vertex":
        return 8 * W + 48 * m + 16 * P + 28 * n
    if mode == "edge":
        return 28 * W + 52 * m + 12 * n
    return 4 * W + 16 * m + 12 * n


def src_sha() -> str:
    """SHA-256 over libbf's CUDA sources and header (ties a committed ncu profile to the code it measured)."""
    import glob
    import hashlib
    h = hashlib.sha256()
    for p in sorted(glob.glob(os.path.join(ROOT, "paper_1907_08607_b200", "csrc", "*"))) + \
            [os.path.join(ROOT, "include", "bf.h")]:
        h.update(open(p, "rb").read())
    return h.hexdigest()[:16]


def load_profile(cfg: int, mode: str, orient: str):
    """The newest committed ncu --set full summary of the wedge kernels for this config and mode."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_full*.json")), reverse=True):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        if d.get("config") == cfg and d.get("mode") == mode and d.get("orient") == orient:
            d["path"] = os.path.relpath(p, ROOT)
            d["matches"] = d.get("src_sha") == src_sha()
            return d
    return None


def config_dict(a, g, W, rank_kind):
    """The workload; identical in both arms (--impl ours / reference)."""
    return {"workload": CONFIG_DESC[a.config] + f"; exact {a.mode} counts, {rank_kind} ranking",
            "config": a.config, "n_u": g.n_u, "n_v": g.n_v, "m": g.m, "W": W, "ranking": rank_kind,
            "mode": a.mode, "l2": "flushed between timed steps (256 MiB device write)",
            "parallelism": f"dp{a.gpus}: wedge-prefix shares of one replicated ranked CSR, NCCL allreduce of outputs"}


def check_parity(a, g, out_u, out_v, out_e, tot):
    """SHA-256 of this run's outputs against the cached exact oracle outputs."""
    import hashlib
    try:
        ref = json.load(open(os.path.join(ROOT, "tests", "golden", "fullsize_oracle.json"))).get(str(a.config))
    except Exception:
        ref = None
    if not ref:
        return {"status": "no cached oracle hash for this config"}
    sha = lambda t: hashlib.sha256(t.cpu().numpy().view(np.uint64).astype("<u8").tobytes()).hexdigest()
    e_sha = hashlib.sha256(np.ascontiguousarray(g.edges).astype("<u4").tobytes()).hexdigest()
    if e_sha != ref["edges_sha256"]:
        return {"status": "MISMATCH: the generated graph differs from the cached one"}
    got = {"total": int(tot.cpu().numpy().view(np.uint64)[0])}
    want = {"total": ref["total"]}
    if a.mode == "vertex":
        got.update(b_u=sha(out_u[:g.n_u]), b_v=sha(out_v[:g.n_v]))
        want.update(b_u=ref["b_u_sha256"], b_v=ref["b_v_sha256"])
    elif a.mode == "edge":
        got["b_e"] = sha(out_e[:g.m])
        want["b_e"] = ref["b_e_sha256"]
    bad = [k for k in want if got[k] != want[k]]
    return {"status": "sha256 match" if not bad else "MISMATCH: " + ",".join(bad),
            "checked": sorted(want), "against": "tests/golden/fullsize_oracle.json (tools/oracle_cache.py)"}


# ----------------------------------------------------------------------------- main
def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import bfgen
    cfgd = bfgen.CONFIGS[a.config]
    rank_kind = a.rank or cfgd["ranking"][0]

    if a.impl == "reference":
        if rank != 0:
            return 0
        return run_reference(a, rank_kind)

    import torch
    import torch.distributed as dist
    from paper_1907_08607_b200 import bf

    g = bfgen.config_graph(a.config)
    n_u, n_v, m = g.n_u, g.n_v, g.m
    n = n_u + n_v

    # CPU oracle baseline first (rank 0, N = 1 only), before any CUDA work; its W
    # comes from the oracle's own ranking + wedge definition
    cpu_base = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            import oracle
            with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
                W_orc, _ = og.wedges(og.rank(rank_kind))
            cpu_base = oracle_sample(g, W_orc, a.cpu_seconds, a.mode)
            cpu_base.pop("est_full_s", None)
            cpu_base.pop("sample_wall_s", None)
        except Exception as ex:  # the baseline is reported, never required
            cpu_base = {"value": None, "unit": UNIT, "cores": 0, "kind": "oracle", "sample": f"failed: {ex}"}

    from paper_1907_08607_b200 import dist as bfd
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", local if world > 1 else 0)
    comm = bfd.nccl_comm_for_group(dev.index) if world > 1 else None

    stream = torch.cuda.current_stream(dev)
    orient = bf.ORIENTS[a.orient]

    def opts(host: bool):
        o = bf.bf_options_default()
        o.device = dev.index
        o.stream = stream.cuda_stream
        o.orient = orient
        if world > 1:
            o.nccl_comm = comm
            o.world_rank = rank
            o.world_size = world
        o.edges_on_device = 0 if host else 1
        o.outputs_on_device = 0 if host else 1
        return o

    edges_dev = torch.from_numpy(g.edges.view(np.int32)).to(dev)
    out_u = torch.empty(max(n_u, 1), dtype=torch.int64, device=dev)
    out_v = torch.empty(max(n_v, 1), dtype=torch.int64, device=dev)
    out_e = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    tot = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(host_bufs=None):
        h = bf.bf_graph_create(n_u, n_v, edges_dev if host_bufs is None else host_bufs["edges"],
                               opts(host_bufs is not None))
        try:
            bf.bf_rank(h, rank_kind)
            if host_bufs is None:
                ou, ov, oe, t = out_u, out_v, out_e, tot
            else:
                ou, ov, oe, t = host_bufs["u"], host_bufs["v"], host_bufs["e"], host_bufs["t"]
            if a.mode == "vertex":
                bf.bf_count_vertex(h, ou, ov, t)
            elif a.mode == "edge":
                bf.bf_count_edge(h, oe, t)
            else:
                bf.bf_count_total(h, t)
            kms, cms, pairs = bf.bf_last_stats(h)
            return dict(W=bf.bf_wedge_count(h), kernel_ms=kms, count_ms=cms, pairs=pairs,
                        launches=bf.bf_launch_count(h), shares=bf.bf_rank_shares(h, world) if world > 1 else None)
        finally:
            bf.bf_graph_destroy(h)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[dev.index])

    # warm-up
    info = None
    for _ in range(max(a.warmup, 0)):
        info = step()
    torch.cuda.synchronize(dev)
    info = info or step()
    W = info["W"]
    shares = info["shares"]

    # timed region (device-resident inputs)
    times, kms, cms, launches, pairs = [], [], [], 0, []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        clk.wait_first()  # nvidia-smi is up and sampling
        for _ in range(a.steps):
            flush.fill_(1)  # L2 flush between timed steps (256 MiB > 126 MB L2)
            torch.cuda.synchronize(dev)
            barrier()
            h0 = time.time()
            ev0.record(stream)
            r = step()
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            clk.timed(h0, time.time())
            times.append(ev0.elapsed_time(ev1))
            kms.append(r["kernel_ms"])
            cms.append(r["count_ms"])
            launches += r["launches"]
            pairs.append(r["pairs"])
    t_local = float(sum(times))
    t_kernel_local = float(np.mean(kms)) if kms else 0.0
    t_count_local = float(np.mean(cms)) if cms else 0.0
    t_max, t_kernel, t_count = bfd.max_over_ranks([t_local, t_kernel_local, t_count_local], device=dev)
    ms_step = t_max / max(a.steps, 1)

    # self-check: the last step's outputs against the cached oracle SHA-256s
    # (tests/golden/fullsize_oracle.json, written by tools/oracle_cache.py from oracle/ only)
    parity = check_parity(a, g, out_u, out_v, out_e, tot)

    # end-to-end through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not a.no_e2e:
        hb = {"edges": torch.from_numpy(g.edges.view(np.int32)).pin_memory().numpy().view(np.uint32),
              "u": torch.empty(max(n_u, 1), dtype=torch.int64).pin_memory().numpy().view(np.uint64),
              "v": torch.empty(max(n_v, 1), dtype=torch.int64).pin_memory().numpy().view(np.uint64),
              "e": torch.empty(max(m, 1), dtype=torch.int64).pin_memory().numpy().view(np.uint64),
              "t": torch.zeros(1, dtype=torch.int64).pin_memory().numpy().view(np.uint64)}
        step(hb)
        et = []
        for _ in range(a.steps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            barrier()
            ev0.record(stream)
            step(hb)
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            et.append(ev0.elapsed_time(ev1))
        te = bfd.max_over_ranks([float(sum(et))], device=dev)[0]
        d2h = {"vertex": 8 * (n_u + n_v) + 8, "edge": 8 * m + 8, "total": 8}[a.mode]
        e2e = {"value": W * a.steps / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * m,
               "d2h_bytes_per_step": d2h, "ms_per_step": te / a.steps}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    value = W * a.steps / (t_max / 1e3)
    P = int(np.median(pairs)) if pairs else 0
    abytes = algorithmic_bytes(a.mode, W, m, n, P)
    if world > 1:  # rank 0's share (its wedges from the plan's deal; slots/vertices pro rata)
        f0 = shares[0] / max(W, 1) if shares else 1.0 / world
        abytes = algorithmic_bytes(a.mode, int(W * f0), int(m * f0), int(n * f0), P)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    if not peak:
        peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    achieved = abytes / (t_kernel / 1e3) / 1e9 if t_kernel > 0 else None
    orient_name = a.orient if a.orient != "auto" else "high"
    prof = load_profile(a.config, a.mode, orient_name)
    traffic = prof.get("dram_bytes_per_launch") if prof else None
    cfg = config_dict(a, g, W, rank_kind)
    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32/u64",
        "data": "synthetic",
        "config": cfg,
        "step": "bf_graph_create + bf_rank + bf_count_* + destroy (SURVEY 8(a) a1-a9), edges resident in HBM",
        "edges_per_s": m * a.steps / (t_max / 1e3),
        "phases_ms": {"t_count": t_count, "t_prep_and_destroy": ms_step - t_count,
                      "note": "t_count = the whole bf_count_* call (CUDA events on the graph's stream, SURVEY 8(d)); "
                              "t_prep = create + rank (ingest, ranking, ranked CSR, plan) + destroy"},
        "count_only": {"kernel_ms": t_kernel, "wedges_per_s": W / (t_kernel / 1e3) if t_kernel else None,
                       "edges_per_s": m / (t_kernel / 1e3) if t_kernel else None,
                       "call_wedges_per_s": W / (t_count / 1e3) if t_count else None,
                       "note": "kernel_ms: the wedge kernels alone (CUDA events around their launches on the "
                               "graph's stream); call = t_count"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "frac_basis": "ALGORITHMIC bytes (SURVEY 8(d) model) / wedge-kernel time / measured HBM copy "
                                   "peak; most re-reads hit L2, so actual DRAM traffic is far lower",
                     "kernel": "wedge kernels (k_split_walk/k_split_finalize, k_big, k_small x2) of one bf_count call",
                     "algorithmic_bytes": abytes, "P_pairs": P,
                     "bytes_model": {"vertex": "8W+48m+16P+28n", "edge": "28W+52m+12n",
                                     "total": "4W+16m+12n"}[a.mode],
                     "peak_source": peak_src},
        "cpu_baseline": cpu_base,
        "e2e": e2e,
        "parity": parity,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if prof:
        dram_gbs = traffic / (prof["kernel_ms"] / 1e3) / 1e9 if traffic and prof.get("kernel_ms") else None
        # instruction-issue ceiling: 4 warp schedulers per SM, one warp instruction each per cycle
        clk_mhz = peaks.get("sm_max_mhz") or 1965.0
        issue_peak = 148 * 4 * clk_mhz * 1e6
        wipw = prof.get("warp_inst_per_wedge")
        issue_rate = wipw * W / (t_kernel / 1e3) if wipw and t_kernel else None
        out["roofline"]["measured"] = {
            "source": prof["path"], "src_sha": prof.get("src_sha"), "matches_this_build": prof.get("matches"),
            "dram_bytes_per_launch": traffic, "dram_gbs": dram_gbs,
            "dram_frac": dram_gbs / peak if dram_gbs else None, "l2_hit_pct": prof.get("l2_hit_pct"),
            "issue_active_pct": prof.get("issue_active_pct"), "warp_inst_per_wedge": wipw,
            "issue_rate_warp_inst_per_s": issue_rate, "issue_peak_warp_inst_per_s": issue_peak,
            "issue_frac": issue_rate / issue_peak if issue_rate else None,
            "issue_basis": "the capture's warp instructions per wedge x W / this run's wedge-kernel time, against "
                           "148 SMs x 4 schedulers x max SM clock",
            "limiter": prof.get("limiter")}
        if not prof.get("matches"):
            out["roofline"]["traffic"] = None  # the profile is of other code: report it beside, not as this run's
    if world > 1:
        out["shares"] = {"wedges_per_rank": shares, "max_over_mean": max(shares) * world / max(sum(shares), 1)}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_reference(a, rank_kind):
    """The reference arm: the CPU oracle as it stands, on the box's host cores,
    each step a bounded sample of the same workload; W from the oracle's own
    ranking and wedge-count definition (not from the GPU path)."""
    import bfgen
    import oracle
    g = bfgen.config_graph(a.config)
    with oracle.OracleGraph(g.n_u, g.n_v, g.edges) as og:
        W, _ = og.wedges(og.rank(rank_kind))
    per_step = max(2.0, min(a.cpu_seconds, 150.0 / max(1, a.steps + a.warmup)))
    vals, fulls, last = [], [], None
    for i in range(a.warmup + a.steps):
        r = oracle_sample(g, W, per_step, a.mode)
        if i >= a.warmup:
            vals.append(r["value"])
            fulls.append(r["est_full_s"])
            last = r
    value = float(np.median(vals))
    ms = float(np.median(fulls)) * 1e3
    out = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": config_dict(a, g, W, rank_kind),
        "ms_per_step_note": "extrapolated: each step times the oracle on a bounded sample of the workload "
                            "(see cpu_baseline.sample) and scales by the oracle's step count",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
