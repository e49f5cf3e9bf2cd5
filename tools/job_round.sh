# round measurements: GPU tests, smoke, bench, sweep, MH chain, launch list, ncu (TAG=rNN)
TAG=${TAG:-r02c}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/gputests_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gputests_$TAG.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
SWEEP_N=${SWEEP_N:-2000,10000,20000,50000,85000,250000,1000000} timeout 900 python tools/sweep.py > gpurun_out/sweep_$TAG.json 2> gpurun_out/sweep_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > /dev/null 2>&1
TAG=$TAG bash tools/run_ncu.sh > /dev/null 2>&1
ls gpurun_out | grep $TAG
