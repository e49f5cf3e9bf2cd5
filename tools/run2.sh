set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -x -q -m gpu 2>&1 | tail -5
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -3 gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r01.json 2>&1; cat gpurun_out/bench_ref_r01.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 -o gpurun_out/prof_pair_r01 python tools/profile_one.py > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
ls -la gpurun_out
