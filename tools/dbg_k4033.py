import sys; sys.path.insert(0,'.')
import bfgen, numpy as np
from paper_1907_08607_b200 import bf
g=bfgen.complete(40,33)
with bf.ButterflyGraph(g.n_u,g.n_v,g.edges,rank="degree",orient="high") as bg:
    print(bg.total())
