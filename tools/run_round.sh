# full round check: GPU tests, smoke, bench (TAG=rNN), outputs in gpurun_out/
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} --durations=25 2>&1 | tail -60 > gpurun_out/gputests_$TAG.txt
tail -5 gpurun_out/gputests_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
