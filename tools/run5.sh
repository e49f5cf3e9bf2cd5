python -m pytest tests -q -m gpu 2>&1 | grep -E "passed|failed|Error|assert" | head -20
bash tools/mh_bench.sh
