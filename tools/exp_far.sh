run() { echo "== $1 $2"; STHK_LIB=$1 QP_SCHED=$2 QP_DENSE=0 QP_MODES=1 timeout 200 python tools/quick_perf.py 2>&1 | grep "grad=1" | awk '{print $1, $6, $7}'; }
L=paper_2005_10123_b200/libsthk.so
run $L 1,2,4
run $L 1,2,6
run $L 1,2,3
run $L 1,1,6
run $L 0,3,6
run tools/variants/libsthk_far4.so 0,3,4
run tools/variants/libsthk_far5.so 0,3,5
run tools/variants/libsthk_far5.so 1,2,5
