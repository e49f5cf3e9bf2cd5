"""BASELINE configs C3 (N sweep 10k-250k) and C4 (N=1M) on one B200:
loglik+gradient, device-timed full evaluations (background cache off),
generateBenchmarkCloud(N, {0,15,0,15,4750}, Rng(N)) at Theta_post and
Theta_init. Prints one JSON document."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402
import bench  # noqa: E402

sizes = [int(v) for v in os.environ.get("SWEEP_N", "10000,20000,50000,85000,100000,150000,200000,250000,1000000").split(",")]
eng = pk.Engine((0,))
eng.set_timing(True)
eng.set_background_cache(False)
peak, _ = bench.eng_peak(pk, 0)
rows = []
for n in sizes:
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
    eng.load(ev)
    for name, th in (("post", bench.THETA_POST), ("init", bench.THETA_INIT)):
        eng.set_params(th)
        reps = 10 if n <= 250000 else 3
        for _ in range(2):
            eng.loglik_grad()
        ev_ms, pk_ms = [], []
        # whole-evaluation device time without events between the kernels
        # (timing level 2), then the pair phase alone (level 1)
        eng.set_timing(2)
        for _ in range(reps):
            r = eng.loglik_grad()
            st = eng.stats()
            ev_ms.append(st["eval_ms"])
        eng.set_timing(1)
        for _ in range(reps):
            eng.loglik_grad()
            pk_ms.append(eng.stats()["pair_kernel_ms"])
        st = eng.stats()
        flops = bench.strict_flops(st)
        t = float(np.median(ev_ms))
        tp = float(np.median(pk_ms))
        row = {"n": n, "theta": name, "eval_ms": t, "pair_kernel_ms": tp, "evals_per_s": 1e3 / t,
               "pair_interactions_per_s_dense_equiv": n * n / (t * 1e-3),
               "ordered_bg_pairs": st["pairs_bg"], "trigger_pairs": st["pairs_tr"],
               "executed_tflops": flops / (tp * 1e-3) / 1e12,
               "roofline_frac_executed": flops / (tp * 1e-3) / 1e12 / peak,
               "roofline_frac_whole_eval": flops / (t * 1e-3) / 1e12 / peak,
               "loglik": r[0], "valid": r[1]}
        rows.append(row)
        print(json.dumps(row), flush=True)
print(json.dumps({"fp64_peak_tflops_measured": peak, "rows": rows}))
