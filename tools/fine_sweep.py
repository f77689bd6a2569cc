"""Fine-grid companion timing sweep (development aid; bench.py is the
contract): one JSON line per (config, S) with ms/step and HBM fraction."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="c3:64,c3:1,c5:1,c5:8")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
for spec in args.cases.split(","):
    cfg, S = spec.split(":")
    r = bench.fine_companion(cfg, int(S), 0, args.steps, 2)
    print(json.dumps({"config": cfg, "S": int(S), "sc": os.environ.get("MSW_FINE_SC", "auto"),
                      "ms_step": r["ms_per_step"], "frac": r["roofline"]["frac"],
                      "unstable": r["unstable_step"]}), flush=True)
