for v in bg5; do echo "== $v"; STHK_LIB=tools/variants/libsthk_$v.so QP_DENSE=0 QP_MODES=1 timeout 200 python tools/quick_perf.py 2>&1 | grep "grad=1" | awk '{print $1, $6, $7}'; done
echo "== base"; QP_DENSE=0 QP_MODES=1 timeout 200 python tools/quick_perf.py 2>&1 | grep "grad=1" | awk '{print $1, $6, $7}'
