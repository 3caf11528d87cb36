"""Re-run chosen triage cases (tools/dbg_triage.py) by substring of their JSON spec, each in a fresh
process, N times:  BF_LIB=libbf_debug.so python tools/dbg_case.py '"rank": "auto"' 5"""
import json, subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import dbg_triage as t

pat, reps = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
cases = [dict(g=["C", 1500, 900, 12000, 2.0, 2.3, 5], mode=m, flags=[], orient="high", rank=r)
         for r in ("side", "approx_degree", "approx_codegen", "auto") for m in ("vertex", "edge")]
n = {}
for c in cases:
    if pat not in json.dumps(c):
        continue
    for _ in range(reps):
        r = subprocess.run([sys.executable, "-c", t.CHILD, json.dumps(c)], capture_output=True, text=True, timeout=180)
        out = r.stdout + r.stderr
        res = "ok" if "RESULT ok" in out else ("mismatch" if "RESULT mismatch" in out else "ERROR")
        print(res, json.dumps(c), " | ".join(l for l in out.splitlines() if "BFError" in l)[:200], flush=True)
        n[res] = n.get(res, 0) + 1
print("SUMMARY", json.dumps(n))
