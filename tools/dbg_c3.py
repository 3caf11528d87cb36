"""Repeat one scaled-config count several times against the oracle (race hunting)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bfgen, oracle, numpy as np
from paper_1907_08607_b200 import bf
k, scale, orient = int(sys.argv[1]), float(sys.argv[2]), sys.argv[3]
flags = 0
for f in sys.argv[4:]:
    flags |= getattr(bf, "BF_FLAG_" + f)
g = bfgen.config_graph(k, scale)
ref = oracle.count(g.n_u, g.n_v, g.edges, edge=False)
rank = bfgen.CONFIGS[k]["ranking"][0]
for rep in range(4):
    with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=rank, orient=orient, test_flags=flags) as bg:
        t = bg.total()
        bu, bv_, t2 = bg.vertex()
    print(rep, t == ref["total"], t2 == ref["total"], np.array_equal(bu, ref["b_u"]), np.array_equal(bv_, ref["b_v"]), t - ref["total"])
