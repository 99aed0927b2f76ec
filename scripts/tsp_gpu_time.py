"""Time the TSP-baseline tours on the GPU at config-5 scale (one CTA per
problem; problem b: points q.sample(1000, [b, 2]), seed b, budget 10 n).

    python scripts/tsp_gpu_time.py [problems]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import tsp  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
q = fc.benchmark_mixture(2)
probs = [(q.sample(1000, [b, 2]), b, None) for b in range(B)]
tsp.build_tours(probs[:2])  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
tours = tsp.build_tours(probs)
dt = time.perf_counter() - t0
print(json.dumps({"what": "GPU tours (nearest neighbour + first-improving 2-opt), config-5 point sets",
                  "problems": B, "seconds": dt, "problems_per_s": B / dt,
                  "mean_length": sum(t.length for t in tours) / B}))
