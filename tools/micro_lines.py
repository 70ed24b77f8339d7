"""Run single bench.py micro lines (cfg4 / cfg5 / cfg3 / cfg1) on one GPU and print them as
JSON -- for iterating on one kernel without the whole bench.
  python tools/micro_lines.py cfg4 cfg5"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_0911_4498_b200 as P  # noqa: E402

ctx = bench.Ctx(0, 1)
peak = 6530.0
fns = {"cfg4": bench.micro_matvec, "cfg5": bench.micro_hankelize, "cfg3": bench.micro_decompose_cfg3,
       "cfg1": lambda P, peak, ctx: bench.micro_decompose_cfg1(P, ctx)}
for w in sys.argv[1:] or ["cfg4", "cfg5"]:
    r = fns[w](P, peak, ctx)
    print(w, json.dumps(r), flush=True)
