"""cfg5 Hankelization: bench line for several four-step batch sizes (SSA_HANK_PER), one process.
  python tools/cfg5_sweep.py 4 8 16 32 64"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_0911_4498_b200 as P  # noqa: E402

ctx = bench.Ctx(0, 1)
for per in sys.argv[1:] or ["8", "16", "32", "64"]:
    os.environ["SSA_HANK_PER"] = per
    r = bench.micro_hankelize(P, 6530.0, ctx)
    print(per, round(r["value"]), round(r["ms"], 2), round(r["roofline"]["frac"], 3), flush=True)
