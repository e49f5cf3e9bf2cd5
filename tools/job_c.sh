{
QP_REPS=60 python tools/perf_matrix.py
STHK_ITEM_TRACE=400000 python tools/item_trace.py c2 post | grep -v "in flight\|stages"
STHK_ITEM_TRACE=400000 python tools/item_trace.py c2 init | grep -v "in flight\|stages"
SWEEP_N=10000,250000,1000000 python tools/sweep.py 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for r in d['rows']: print(r['n'], r['theta'], round(r['eval_ms']*1e3,1), round(r['pair_kernel_ms']*1e3,1))"
timeout 1500 python -m pytest tests -q -m gpu -x -k "not c4_1m" 2>&1 | tail -3
} > gpurun_out/c.txt 2>&1
