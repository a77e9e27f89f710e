"""Run one scaling-sweep variant (tools/sweep.py names) once and report the outcome.

    python tools/probe_variant.py indoor_n4000_N16
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import sweep  # noqa: E402
from paper_1607_06886_b200 import api  # noqa: E402

want = sys.argv[1]
for name, sc in list(sweep.variants("scaling")) + list(sweep.variants("named")):
    if name != want:
        continue
    ctx = api.Context(0)
    t = time.time()
    try:
        r = api.run_pump(api.parse_scenario(json.dumps(sc)), ctx=ctx)
        print(name, "ok", round(time.time() - t, 3), "s", {k: r[k] for k in ("success", "partial_plans", "cost")})
    except Exception as e:  # report, do not hide: this is a probe
        print(name, "FAILED", type(e).__name__, str(e)[:300])
