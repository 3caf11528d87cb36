"""Per-rank wedge shares of the multi-GPU deal for BASELINE.json's
configs at G = 2, 4, 8: bf_rank_shares reports, from the plan the library
builds, the wedges each rank's kernels would process (split starts whole in
snake order, tier segments through bf_deal_index).  Prints max/mean per G and
the largest single start's share of W (the bound on whole-start dealing).

  python tools/rank_shares.py [k ...] > gpurun_out/rank_shares.json   (needs a GPU)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bfgen  # noqa: E402
from paper_1907_08607_b200 import bf  # noqa: E402


def main(ks):
    out = {}
    for k in ks:
        g = bfgen.config_graph(k)
        rank = bfgen.CONFIGS[k]["ranking"][0]
        with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank) as bg:
            W = bg.wedges()
            ws = bg.export_csr()["wstart"]
            top = int(ws.max()) if len(ws) else 0
            row = {"W": W, "ranking": rank, "largest_start_share": top / max(W, 1)}
            for G in (2, 4, 8):
                sh = bf.bf_rank_shares(bg.h, G)
                assert sum(sh) == W
                row[f"G{G}"] = {"max_over_mean": max(sh) * G / max(W, 1), "wedges_per_rank": sh}
        out[f"c{k}"] = row
        print(json.dumps({f"c{k}": {kk: (v if not isinstance(v, dict) else v["max_over_mean"])
                                    for kk, v in row.items()}}), flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "rank_shares.json"), "w"), indent=1)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [2, 3, 4, 5])
