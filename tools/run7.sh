for v in g4_m3 g4_m2 g2_m3 g2_m4; do echo "== $v"; STHK_LIB=tools/variants/libsthk_$v.so QP_MODES=1 QP_DENSE=0 timeout 300 python tools/quick_perf.py 2>&1 | grep -E "grad"; done
