"""Run one stream fixture (debugging aid: use under compute-sanitizer)."""
import sys
sys.path.insert(0, ".")
from oracle import fixtures
from paper_1810_08061_b200 import ir
from paper_1810_08061_b200.executor import execute_stream
from paper_1810_08061_b200 import stream as st

name = sys.argv[1] if len(sys.argv) > 1 else "lbfgs_m3_n50"
doc = fixtures.load_golden(name)
g = ir.from_json(doc["graph"])
res = execute_stream(g, fixtures.make_stream_feeds(doc["case"]))
print(st.run.last)
for o in res.outputs:
    print(getattr(o, "shape", None), getattr(o, "array", o) if getattr(o, "shape", (1,)) == () else "")
print("expected", [o["tensor"]["data"][:3] for o in doc["expected"].get("outputs", [])])
