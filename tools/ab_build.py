"""Build A/B variants of the library with -D macros into _ab/<name>.so:
   python tools/ab_build.py name1:DEF=1,DEF2=3 name2:DEF=2 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_01579_b200 import build
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "_ab")
os.makedirs(root, exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    out = os.path.join(root, name + ".so")
    print(build.build(out=out, defs=[d for d in defs.split(",") if d]))
    import shutil
    shutil.rmtree(out + ".objs", ignore_errors=True)
