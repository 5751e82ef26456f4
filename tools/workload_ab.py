"""Time one bench.SWEEP workload (name substring) and print ms/step, roofline
fraction and per-kernel device times (A/B runs: set SKL_* switches in the env)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_15473_b200 as skl  # noqa: E402

name = sys.argv[1]
c = [c for c in bench.SWEEP + [("c2 bf16", 768, 3072, 2, 128, 32768, "bf16")] if name in c[0]][0]
graph = os.environ.get("GRAPH", "0") == "1"  # replay the step from a CUDA graph (launch-bound shapes)
r = bench.measure_workload(skl, torch, torch.device("cuda", 0), *c, steps=20, warmup=5, graph=graph)
skl.profile_enable(True)
skl.profile_collect()
bench.measure_workload(skl, torch, torch.device("cuda", 0), *c, steps=5, warmup=1)
prof = skl.profile_collect()
print(json.dumps({"workload": c[0], "env": {k: v for k, v in os.environ.items() if k.startswith("SKL_")},
                  "ms_per_step": round(r["ms_per_step"], 4), "ms_per_step_eager": round(r["ms_per_step_eager"], 4), "roofline_frac": round(r["roofline_frac"], 4),
                  "kernels_us": {k: round(t / n * 1e3, 1) for k, (n, t) in prof.items()}}))
