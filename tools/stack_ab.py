"""c5 stack step (graph replay) under the current SKL_* env: ms per step (A/B of switches)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_15473_b200 as skl  # noqa: E402

r = bench.measure_stack(skl, torch, torch.device("cuda", 0), 1, steps=10, warmup=3)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SKL_")},
                  "ms_per_step": round(r["ms_per_step"], 4), "roofline_frac": round(r["roofline_frac"], 4)}))
