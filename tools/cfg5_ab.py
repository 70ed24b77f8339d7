"""cfg5 Hankelization A/B in one process: the bench line with an environment knob of the
long path unset / set, interleaved (same box, same clocks).
  python tools/cfg5_ab.py SSA_ROW_MINB3 [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_0911_4498_b200 as P  # noqa: E402

knob = sys.argv[1] if len(sys.argv) > 1 else "SSA_ROW_MINB3"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = bench.Ctx(0, 1)
for r in range(rounds):
    for on in (0, 1):
        if on:
            os.environ[knob] = "1"
        else:
            os.environ.pop(knob, None)
        m = bench.micro_hankelize(P, 6530.0, ctx)
        print(knob, on, round(m["value"]), round(m["ms"], 2), round(m["roofline"]["frac"], 3), flush=True)
