"""Short driver for ncu captures: C2 workload, a few loglik+grad evaluations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402

theta = bench.THETA_INIT if "--init" in sys.argv else bench.THETA_POST
x, y, t, T = bench.make_workload()
e = pk.Engine((0,))
e.load_events(x, y, t, T)
e.set_params(theta)
e.set_background_cache(False)  # every launch a full sweep
for _ in range(5):
    r = e.loglik_grad()
print("loglik", r[0])
