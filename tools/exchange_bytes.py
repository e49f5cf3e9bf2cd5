"""fx bytes the owner-directed exchange moves per evaluation (k emulated ranks
on one GPU, full sweeps): C2 and C4 (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_10123_b200 as pk  # noqa: E402

TH = [0.66, 1.6, 14, 0.344, 1440, 0.0695]
c2 = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                               pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=85000)[0]
c4 = pk.generateBenchmarkCloud(1000000, pk.SimWindow(0, 15, 0, 15, 4750), 1000000)
for name, ev in (("C2", c2), ("C4", c4)):
    for k in (2, 4, 8):
        with pk.Engine((0,) * k) as e:
            e.load(ev)
            e.set_background_cache(False)
            e.set_params(TH)
            e.loglik_grad()
            b = e.exchange_bytes()
            print(f"{name} N={ev.size()} ranks={k}: {b} B total, {b / (k - 1):.0f} B per sending rank, "
                  f"allreduce of fx would move {6 * 8 * ev.size()} B per rank", flush=True)
