"""Host wall-clock breakdown of one bench step (create / rank / count / destroy)
on a config, device-resident edges, after warm-up."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bfgen
from paper_1907_08607_b200 import bf
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = bfgen.config_graph(k)
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
e = torch.from_numpy(g.edges.view(np.int32)).to(dev)
ou = torch.empty(g.n_u, dtype=torch.int64, device=dev); ov = torch.empty(g.n_v, dtype=torch.int64, device=dev)
t = torch.zeros(1, dtype=torch.int64, device=dev)
rank = bfgen.CONFIGS[k]["ranking"][0]
for rep in range(5):
    o = bf.bf_options_default(); o.stream = s.cuda_stream; o.edges_on_device = 1; o.outputs_on_device = 1
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = bf.bf_graph_create(g.n_u, g.n_v, e, o); torch.cuda.synchronize(); t1 = time.perf_counter()
    bf.bf_rank(h, rank); torch.cuda.synchronize(); t2 = time.perf_counter()
    bf.bf_count_vertex(h, ou, ov, t); torch.cuda.synchronize(); t3 = time.perf_counter()
    kms, cms, _ = bf.bf_last_stats(h)
    bf.bf_graph_destroy(h); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.3f} rank {1e3*(t2-t1):.3f} count {1e3*(t3-t2):.3f} (kernels {kms:.3f}, call {cms:.3f}) destroy {1e3*(t4-t3):.3f} total {1e3*(t4-t0):.3f} ms")
