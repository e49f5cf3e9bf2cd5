run() { echo "== $1"; QP_SCHED=$1 QP_DENSE=0 QP_MODES=1 timeout 200 python tools/quick_perf.py 2>&1 | grep "grad=1" | awk '{print $1, $6, $7}'; }
run 1,3,6
run 3,3,6
run 3,3,3
run 2,3,6
run 0,3,6
