"""A few full loglik+grad evaluations of an N-event cloud (env SN, default
10000) with the sweep caches off: the workload for an ncu launch list of the
small-N path (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_10123_b200 as pk  # noqa: E402

n = int(os.environ.get("SN", "10000"))
e = pk.Engine((0,))
e.set_background_cache(False)
ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
e.load(ev)
e.set_params([0.66, 1.6, 14, 0.344, 1440, 0.0695])
for _ in range(int(os.environ.get("SREP", "5"))):
    print(e.loglik_grad()[0])
