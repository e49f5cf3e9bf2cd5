{
for v in "1 1" "0 1" "1 0" "0 0"; do set -- $v
echo "== STHK_EV1_NODE=$1 STHK_NODE_PRIO=$2"
STHK_EV1_NODE=$1 STHK_NODE_PRIO=$2 python bench.py --steps 300 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['e2e']['value'], d['roofline']['pair_kernel_ms'])"
STHK_EV1_NODE=$1 STHK_NODE_PRIO=$2 STHK_ITEM_TRACE=400000 python tools/item_trace.py c2 post | grep -A9 timeline | grep "plan \|trigger\|far \|general \|finalize"
STHK_EV1_NODE=$1 STHK_NODE_PRIO=$2 STHK_ITEM_TRACE=400000 python tools/item_trace.py c2 init | grep -A9 timeline | grep "plan \|trigger\|far \|general \|finalize"
done
} > gpurun_out/c.txt 2>&1
