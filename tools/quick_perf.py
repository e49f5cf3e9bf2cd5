"""Quick timing probe (not the bench contract): C2 data at both thetas, both
pair-kernel variants, culled and dense."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402

N = int(os.environ.get("QP_N", "85000"))
ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                  pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=N)
e = pk.Engine((0,))
e.load(ev)
e.set_timing(True)
e.set_background_cache(bool(int(os.environ.get("QP_CACHE", "0"))))
e._lib.sthk_set_far_tier(e._h, int(os.environ.get("QP_FAR", "1")))
if "QP_SCHED" in os.environ:  # concurrent,near_ctas,far_ctas
    c, nc, fc = (int(v) for v in os.environ["QP_SCHED"].split(","))
    e._lib.sthk_set_far_schedule(e._h, c, nc, fc)
modes = [int(m) for m in os.environ.get("QP_MODES", "0,1").split(",")]
denses = [bool(int(d)) for d in os.environ.get("QP_DENSE", "0,1").split(",")]
for name, p in [("post", [0.66, 1.6, 14, 0.344, 1440, 0.0695]), ("init", [1, 1.6, 14, 0.1, 1, 1])]:
    e.set_params(p)
    for mode in modes:
        e.set_kernel(mode)
        for dense in denses:
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
                g = r[2] if grad else None
                print(f"{name} mode={mode} dense={int(dense)} grad={int(grad)} ll={r[0]:.12f} "
                      f"wall_ms={1e3*np.median(ts):.3f} pair_ms={st['pair_kernel_ms']:.3f} "
                      f"eval_ms={st['eval_ms']:.3f} sc={st['source_chunk']} bg={st['pairs_bg']:.3e} "
                      f"tr={st['pairs_tr']:.3e} xbg={st['exec_bg']:.3e} xsym={st['exec_sym']:.3e} xfar={st['exec_far']:.3e}"
                      + (f" g0={g[0]:.12e} g5={g[5]:.12e}" if grad else ""), flush=True)
