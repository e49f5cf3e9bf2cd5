"""MH-style moves on C2 data for an ncu capture of the cached-background
paths (development tool): env MOVE = h | omega | mu0, N (default 85000).
Only the last REP moves are inside cudaProfilerStart/Stop, so run ncu with
--profile-from-start off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402

n = int(os.environ.get("N", "85000"))
move = {"mu0": 0, "h": 5, "omega": 4}[os.environ.get("MOVE", "h")]
ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                  pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=n)
e = pk.Engine((0,))
e.load(ev)
p = np.array([0.66, 1.6, 14, 0.344, 1440, 0.0695])
e.set_params(p)
e.loglik()
for i in range(6):
    p[move] *= 1.01 if i % 2 else 1 / 1.01
    e.set_params(p)
    e.loglik()
torch.cuda.profiler.start()
for i in range(int(os.environ.get("REP", "2"))):
    p[move] *= 1.01 if i % 2 else 1 / 1.01
    e.set_params(p)
    print(e.loglik()[0], e.stats()["cache_hit"], e.stats()["work_items"])
torch.cuda.profiler.stop()
