set -x
python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()"
timeout 300 python tools/quick_perf.py
