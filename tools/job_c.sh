{
for n in c2 10000 250000; do STHK_ITEM_TRACE=400000 python tools/item_trace.py $n post | grep -A4 timeline; done
QP_REPS=60 python tools/perf_matrix.py
SN=2000,10000,20000 python tools/small_n.py 2>&1 | grep cloud
timeout 1500 python -m pytest tests -q -m gpu -x -k "not c4_1m" 2>&1 | tail -3
} > gpurun_out/c.txt 2>&1
