"""Timing matrix for kernel variants / schedules (development tool).
C2 loglik+grad at Theta_post and Theta_init, device eval time (engine timing
events), median of REPS evaluations. Run once per library variant:
  STHK_LIB=tools/variants/libsthk_X.so python tools/perf_matrix.py [sched ...]
where each sched is "concurrent,near_ctas,far_ctas" (default: engine default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402

N = int(os.environ.get("QP_N", "85000"))
REPS = int(os.environ.get("QP_REPS", "30"))
ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                  pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=N)
e = pk.Engine((0,))
e.load(ev)
e.set_timing(True)
e.set_background_cache(False)
scheds = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [None]
tag = os.path.basename(os.environ.get("STHK_LIB", "default"))
for sc in scheds:
    if sc:
        e.set_far_schedule(*sc)
    for name, p in [("post", [0.66, 1.6, 14, 0.344, 1440, 0.0695]), ("init", [1, 1.6, 14, 0.1, 1, 1])]:
        e.set_params(p)
        for _ in range(3):
            e.loglik_grad()
        ev_ms, pk_ms = [], []
        for _ in range(REPS):
            r = e.loglik_grad()
            st = e.stats()
            ev_ms.append(st["eval_ms"])
            pk_ms.append(st["pair_kernel_ms"])
        print(f"{tag} sched={sc} {name} eval_ms={np.median(ev_ms):.4f} pair_ms={np.median(pk_ms):.4f} "
              f"A={st['far_threshold']:.2f} tfar={st['far_split_days']:.1f} "
              f"ll={r[0]!r} g={r[2][0]!r}", flush=True)
