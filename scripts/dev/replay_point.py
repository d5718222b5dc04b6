"""Replay chosen (system, rhs) points of a C4 device build on the CPU checker (oracle/replay.py)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1602_00138_b200 import build, problem as P
build.build()
import replay as RP
c = P.CONFIGS["C4"]
pts = {int(k): [int(x) for x in v] for k, v in json.loads(sys.argv[1]).items()}
ns = max(pts)
out, smp = RP.run_device_build(c, pts, systems=list(range(1, ns + 1)), seed_check=False, verbose=False)
print(json.dumps({"rows": [[r[0], r[1], r[4], r[5], r[10]] for r in out["rows_detail"]], "maxdiff": out["max_iteration_diff"]}))
