# full ncu captures of the pair kernels of one evaluation (C2, Theta_post):
# the near kernels (trigger-free, general), the far kernel and the row-window trigger kernel
TAG=${TAG:-r01}
ncu -f --set full --clock-control none --import-source on -k regex:"sym_kernel|pair_kernel|far_kernel|trig_rows" -s 6 -c 3 -o gpurun_out/prof_pair_$TAG python tools/profile_one.py > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
ls -la gpurun_out | grep $TAG
