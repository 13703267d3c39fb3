"""Time bench.py's ragged / paged batch (f2) for one config: packed-row K/V
and K/V in a page pool (pages of 16 and 64 keys).  PARSE_LIB picks a library
variant (A/B).

    python tools/time_ragged.py qwen3_235b [--iters 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_04263_b200 as pb  # noqa: E402
import workloads  # noqa: E402
from bench import bench_ragged  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
for name in a.configs:
    r = bench_ragged(pb, workloads.CONFIGS[name], "cuda", 1654.1, iters=a.iters)
    print(json.dumps({"config": name, "lib": os.path.basename(os.environ.get("PARSE_LIB", "libparse.so")),
                      **{k: round(v["ms"], 4) for k, v in r.items() if isinstance(v, dict)}}), flush=True)
