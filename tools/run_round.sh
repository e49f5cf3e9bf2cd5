# full round check: GPU tests, bench, launch list, one full ncu capture of the pair kernel
TAG=${TAG:-r01}
python -m pytest tests -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/gputests_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
TAG=$TAG bash tools/run_bench.sh
