"""Compare the cluster solver with the legacy one (FCB_OT_LEGACY) on small shapes."""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2511_11514_b200 as fc
    rng = np.random.default_rng(0)
    for n, m in [(5, 7), (200, 2000), (1000, 300), (2000, 10000)]:
        X, Y = rng.random((n, 2)), rng.random((m, 2))
        d = fc.sinkhorn_divergence(X, Y)
        ot = fc.entropic_ot(X, Y)
        print(f"{n}x{m} div={d:.10g} f0={float(ot.f[0]):.10g} g0={float(ot.g[0]):.10g} "
              f"iters={ot.iters_used}")
    sys.exit(0)
for leg in ("1", "0"):
    env = dict(os.environ, FCB_OT_LEGACY=leg)
    print("legacy" if leg == "1" else "cluster")
    r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
    print(r.stdout, r.stderr[-2000:])
