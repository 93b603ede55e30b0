"""Single-scan latency (device time per frame, eager and CUDA graph; plus the
host-to-host run_pipeline call) for the library at LSEG_LIB_PATH.
usage: python tools/latency.py [tag]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

res = bench.single_scan_latency(torch.device("cuda", 0))
tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("LSEG_LIB_PATH", "default").rsplit("/", 1)[-1]
print(tag, json.dumps({k: {m: round(v, 1) for m, v in d.items() if m != "points"} for k, d in res.items()}))
