"""Quick timing probe (not the bench contract): C2 data at both thetas."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_10123_b200 as pk

ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                  pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=85000)
e = pk.Engine((0,))
e.load(ev)
e.set_timing(True)
for name, p in [("post", [0.66, 1.6, 14, 0.344, 1440, 0.0695]), ("init", [1, 1.6, 14, 0.1, 1, 1])]:
    e.set_params(p)
    for dense in (False, True):
        e.set_dense(dense)
        for grad in (True, False):
            for _ in range(3):
                r = e.loglik_grad() if grad else e.loglik()
            ts = []
            for _ in range(10):
                t0 = time.perf_counter()
                r = e.loglik_grad() if grad else e.loglik()
                ts.append(time.perf_counter() - t0)
            st = e.stats()
            print(f"{name} dense={dense} grad={grad} ll={r[0]:.10f} wall_ms={1e3*np.median(ts):.3f} "
                  f"pair_ms={st['pair_kernel_ms']:.3f} eval_ms={st['eval_ms']:.3f} sc={st['source_chunk']} "
                  f"bg={st['pairs_bg']:.3e} tr={st['pairs_tr']:.3e} dense={st['pairs_dense']:.3e}", flush=True)
