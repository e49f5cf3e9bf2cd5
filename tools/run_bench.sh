# round bench + launch list + one full ncu capture of the pair kernel
TAG=${TAG:-r01}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sym_kernel|pair_kernel" -s 3 -c 1 -o gpurun_out/prof_pair_$TAG python tools/profile_one.py > /dev/null 2>&1
ls gpurun_out | grep $TAG
