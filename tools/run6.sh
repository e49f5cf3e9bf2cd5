python -m pytest tests -q -m gpu -x 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout 600 python tools/quick_perf.py
