"""Build tuning variants of libbf for an A/B run on one box (tools/ab.sh):
  python tools/ab_build.py name:DEF=1,DEF2=3 name2: ...   (empty defines = the defaults)
Each variant is libbf_<name>.so in the package directory; load it with BF_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_08607_b200 import build as b

for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    b.build(variant=name, defines=tuple(d for d in defs.split(",") if d))
    print("built", name)
