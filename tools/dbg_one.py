"""Run one small case (argv: json spec as in dbg_triage) and print the result."""
import json, subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.dbg_triage import CHILD  # noqa
r = subprocess.run([sys.executable, "-c", CHILD, sys.argv[1]], capture_output=True, text=True, timeout=120)
print(r.stdout[-3000:], r.stderr[-3000:])
