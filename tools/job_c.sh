{
python bench.py --steps 300 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['e2e']['value'], d['roofline']['pair_kernel_ms'], d['loglik'], d['grad'], d['pairs_per_eval'])"
QP_REPS=40 python tools/perf_matrix.py
STHK_ITEM_TRACE=400000 python tools/item_trace.py c2 post | grep -A12 "general "
SN=2000,10000,20000 python tools/small_n.py 2>&1 | grep cloud
timeout 1500 python -m pytest tests -q -m gpu -x -k "not c4_1m" 2>&1 | tail -15
} > gpurun_out/c.txt 2>&1
