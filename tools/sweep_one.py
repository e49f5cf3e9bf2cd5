"""One C3 sweep point (generateBenchmarkCloud(N, Rng(N))) evaluated a few times
at Theta_post: a short driver for ncu launch lists (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_10123_b200 as pk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
e = pk.Engine((0,))
e.load(ev)
e.set_background_cache(False)
e.set_params([0.66, 1.6, 14, 0.344, 1440, 0.0695])
for _ in range(6):
    r = e.loglik_grad()
print("loglik", r[0])
