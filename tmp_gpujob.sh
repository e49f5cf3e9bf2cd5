mkdir -p gpurun_out
ncu -f --set full --clock-control none --import-source on -k regex:"sym_kernel|far_kernel" -s 6 -c 3 -o gpurun_out/prof_r02b_post python tools/profile_one.py > gpurun_out/ncu_r02b_post.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"sym_kernel|far_kernel" -s 4 -c 2 -o gpurun_out/prof_r02b_init python tools/profile_one.py --init > gpurun_out/ncu_r02b_init.log 2>&1
tail -2 gpurun_out/ncu_r02b_*.log
ls -la gpurun_out/
