python -m pytest tests -q -m gpu 2>&1 | grep -E "passed|failed|Error|assert" | head -20
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 -o gpurun_out/prof_pair_r01b python tools/profile_one.py > /dev/null 2>&1
ncu --set full --clock-control none -c 1 -o gpurun_out/prof_dfma_probe ./tools/fp64_peak > /dev/null 2>&1
ls gpurun_out
