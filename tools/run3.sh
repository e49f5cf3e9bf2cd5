python -m pytest tests -q -m gpu 2>&1 | grep -E "passed|failed|Error|assert" | head -20
for v in 4 5 6; do echo "== minb $v"; STHK_LIB=tools/variants/libsthk_minb$v.so timeout 300 python tools/quick_perf.py 2>&1 | grep -E "grad=True"; done
