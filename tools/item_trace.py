"""Per-item timeline of the pair kernels of one evaluation (development
tool; needs STHK_ITEM_TRACE=<entries>): item durations by kernel, stage count
and diagonal flag, the kernel spans, SM busy fraction and the tail.
usage: STHK_ITEM_TRACE=200000 python tools/item_trace.py [N|c2] [post|init]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2005_10123_b200 as pk  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
th = sys.argv[2] if len(sys.argv) > 2 else "post"
theta = [0.66, 1.6, 14, 0.344, 1440, 0.0695] if th == "post" else [1, 1.6, 14, 0.1, 1, 1]
if which == "c2":
    ev, _ = pk.simulateClusterProcess(pk.Params(1, 1.6, 14, 0.344, 1440, 0.0695),
                                      pk.SimWindow(0, 15, 0, 15, 4750), 0.053217, 2005, keep=85000)
else:
    n = int(which)
    ev = pk.generateBenchmarkCloud(n, pk.SimWindow(0, 15, 0, 15, 4750), n)
e = pk.Engine((0,))
move = os.environ.get("IT_MOVE")  # (h / omega / mu0: a cached MH-style move from theta)
e.set_background_cache(move is not None)
e.set_timing(os.environ.get("IT_TIMING", "1") == "1")
e.load(ev)
e.set_params(theta)
for _ in range(5):
    e.loglik_grad()
if move:
    k = {"mu0": 0, "theta": 3, "omega": 4, "h": 5}[move]
    for i in range(5):
        th2 = list(theta)
        th2[k] *= 1.0 + 0.01 * (i + 1)
        e.set_params(th2)
        e.loglik_grad()
st = e.stats()
raw = e.item_trace()
cta = raw[raw[:, 2] == 0xFFFFFFFF]
tr = raw[raw[:, 2] != 0xFFFFFFFF]
print(f"{which} {th}: eval {st['eval_ms'] * 1e3:.1f} us, pair phase {st['pair_kernel_ms'] * 1e3:.1f} us, "
      f"{len(tr)} items, far threshold A {st['far_threshold']:.2f} split {st['far_split_days']:.1f} d")
t00 = raw[:, 5].min()
names = {1: "general", 2: "trigger-free", 3: "far", 4: "plan", 5: "prep", 6: "finalize", 7: "plan:pivots", 8: "plan:ranges", 9: "plan:histogram", 10: "plan:scan", 11: "trig_rows"}
print("  kernel timeline (first CTA start .. last CTA end, us from the first start):")
for k in sorted(set(cta[:, 0].tolist()), key=lambda k: cta[cta[:, 0] == k, 5].min()):
    m = cta[:, 0] == k
    print(f"    {names.get(k, k):12s} {(cta[m, 5].min() - t00) / 1e3:7.1f} .. {(cta[m, 6].max() - t00) / 1e3:7.1f}"
          f"   ({m.sum()} CTAs)")
for k in (2, 1, 3):
    m = tr[:, 0] == k
    if not m.any():
        continue
    d = (tr[m, 6] - tr[m, 5]) / 1e3
    s0, s1 = (tr[m, 5].min() - t00) / 1e3, (tr[m, 6].max() - t00) / 1e3
    sms = len(np.unique(tr[m, 1]))
    busy = d.sum() / (sms * (s1 - s0)) if s1 > s0 else 0
    print(f"  {names[k]:12s} items {m.sum():5d} span {s0:7.1f}..{s1:7.1f} us  SMs {sms}  "
          f"item us: mean {d.mean():6.2f} p50 {np.median(d):6.2f} max {d.max():6.2f}  "
          f"sum {d.sum():8.1f} (per-SM busy {busy:.2f})")
    for stg in np.unique(tr[m, 3]):
        for dg in (0, 1):
            mm = m & (tr[:, 3] == stg) & (tr[:, 4] == dg)
            if mm.sum() == 0:
                continue
            dd = (tr[mm, 6] - tr[mm, 5]) / 1e3
            print(f"      stages {stg:3d} diag {dg}: {mm.sum():5d} items, us mean {dd.mean():6.2f} "
                  f"max {dd.max():6.2f}")
    # tail: when do the last 10% of items end vs the first end
    ends = np.sort(tr[m, 6] - t00) / 1e3
    print(f"      ends: p10 {ends[len(ends) // 10]:.1f} p50 {ends[len(ends) // 2]:.1f} "
          f"p90 {ends[9 * len(ends) // 10]:.1f} max {ends[-1]:.1f} us")
# concurrency profile: items in flight per 2 us bin
if len(tr) == 0:
    sys.exit(0)
t1 = (tr[:, 6].max() - t00) / 1e3
bins = np.arange(0, t1 + 2, 2.0)
line = []
for b in bins:
    live = ((tr[:, 5] - t00) / 1e3 <= b + 1) & ((tr[:, 6] - t00) / 1e3 > b + 1)
    line.append(int(live.sum()))
print("  items in flight per 2 us:", line)
