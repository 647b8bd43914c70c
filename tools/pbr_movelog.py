import os, sys, json, subprocess
sys.path.insert(0, "."); sys.path.insert(0, "tests")
os.environ["MGK_PBR_DEBUG"] = "1"
from conftest import graph_from_json
import paper_1910_06310_b200 as mgk
rec = [r for r in json.load(open("tests/golden/structure.json")) if r["name"] == sys.argv[1]][0]
g = graph_from_json(rec["graph"])
mgk.pbr_reorder_many([g], seed=0)
