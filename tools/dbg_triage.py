"""Run small cases each in a fresh process (CUDA errors are sticky) and report
which (graph, mode, flags) combinations fail.  Debug tool for GPU bring-up."""
import json, subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import sys, json; sys.path.insert(0, ".")
import bfgen, numpy as np, oracle
from paper_1907_08607_b200 import bf
spec = json.loads(sys.argv[1])
if spec["g"][0] == "K": g = bfgen.complete(*spec["g"][1:])
elif spec["g"][0] == "cfg": g = bfgen.config_graph(*spec["g"][1:])
else: g = bfgen.chung_lu(*spec["g"][1:])
ref = oracle.count(g.n_u, g.n_v, g.edges)
f = 0
for name in spec["flags"]: f |= getattr(bf, "BF_FLAG_" + name)
with bf.ButterflyGraph(g.n_u, g.n_v, g.edges, rank=spec["rank"], orient=spec["orient"], test_flags=f) as bg:
    if spec["mode"] == "total": ok = bg.total() == ref["total"]
    elif spec["mode"] == "vertex":
        bu, bv_, t = bg.vertex(); ok = t == ref["total"] and np.array_equal(bu, ref["b_u"]) and np.array_equal(bv_, ref["b_v"])
    else:
        be, t = bg.edge(); ok = t == ref["total"] and np.array_equal(be, ref["b_e"])
print("RESULT", "ok" if ok else "mismatch")
'''

def main():
  cases = []
  counts = {}
  for gspec in (["K", 40, 33], ["K", 17, 9], ["C", 1500, 900, 12000, 2.0, 2.3, 5], ["cfg", 4, 0.01]):
      for mode in ("total", "vertex", "edge"):
          for flags in ([], ["FORCE_WARP"], ["FORCE_CTA"], ["FORCE_DENSE"], ["FORCE_DENSE", "SMALL_CHUNK"], ["SMALL_CHUNK"],
                        ["UNPACKED_SORT"], ["NO_DENSE_ROW"], ["KEY_BUFFER"], ["FORCE_DENSE", "SMALL_CHUNK", "KEY_BUFFER"]):
              for orient in ("high", "low"):
                  cases.append(dict(g=gspec, mode=mode, flags=flags, orient=orient, rank="degree"))
  # other rankings, and repeated runs of one larger graph (a nondeterministic race
  # shows up as a run that differs)
  for rank in ("side", "approx_degree", "approx_codegen", "auto"):
      for mode in ("vertex", "edge"):
          cases.append(dict(g=["C", 1500, 900, 12000, 2.0, 2.3, 5], mode=mode, flags=[], orient="high", rank=rank))
  for rep in range(4):
      for mode in ("total", "vertex", "edge"):
          cases.append(dict(g=["cfg", 3, 0.02], mode=mode, flags=[], orient="high", rank="approx_degree", rep=rep))
  # race stress under the bounds-checking build: pseudo-random grids per launch
  for rep in range(3):
      for gspec, rank in ((["cfg", 3, 0.02], "approx_degree"), (["cfg", 4, 0.01], "degree")):
          for mode in ("total", "vertex", "edge"):
              for flags in (["GRID_JITTER"], ["GRID_JITTER", "SMALL_CHUNK"], ["GRID_JITTER", "SMALL_WINDOW"]):
                  cases.append(dict(g=gspec, mode=mode, flags=flags, orient="high", rank=rank, rep=rep))
  for c in cases:
      try:
          r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(c)], capture_output=True, text=True, timeout=180)
          out = (r.stdout + r.stderr)
      except subprocess.TimeoutExpired:
          out = "TIMEOUT"
      res = "ok" if "RESULT ok" in out else ("mismatch" if "RESULT mismatch" in out else
                                             ("TIMEOUT" if out == "TIMEOUT" else "ERROR"))
      extra = [l for l in out.splitlines() if "BF_CHECK" in l or "BFError" in l][:2]
      print(res, json.dumps(c), " | ".join(extra)[:300], flush=True)
      counts[res] = counts.get(res, 0) + 1
  print("SUMMARY", json.dumps(counts), f"{len(cases)} cases", flush=True)


if __name__ == "__main__":
    main()
