"""Small-N timing (C3 clouds and C2 prefixes): both pair-kernel variants,
device eval time via the engine's timing events (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402

e = pk.Engine((0,))
e.set_timing(True)
e.set_background_cache(False)
for n in [int(v) for v in os.environ.get("SN", "2000,5000,10000,20000,50000").split(",")]:
    for kind in ("cloud", "c2"):
        if kind == "cloud":
            ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
        else:
            ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                              pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=n)
        e.load(ev)
        for th in ([0.66, 1.6, 14, 0.344, 1440, 0.0695], [1, 1.6, 14, 0.1, 1, 1]):
            e.set_params(th)
            out = []
            for mode in (1, 0):
                e.set_kernel(mode)
                for _ in range(3):
                    e.loglik_grad()
                ev_ms, pk_ms = [], []
                for _ in range(15):
                    e.loglik_grad()
                    st = e.stats()
                    ev_ms.append(st["eval_ms"])
                    pk_ms.append(st["pair_kernel_ms"])
                out.append(f"mode{mode} eval {np.median(ev_ms) * 1e3:7.1f} us pair {np.median(pk_ms) * 1e3:7.1f} us")
            e.set_kernel(1)
            print(f"N={n:6d} {kind:5s} th={'post' if th[4] > 100 else 'init'}  " + "  |  ".join(out), flush=True)
