# one full ncu capture of the far-tier kernel (C2, Theta_post)
TAG=${TAG:-r01}
ncu --set full --clock-control none --import-source on -k regex:"far_kernel" -s 3 -c 1 -o gpurun_out/prof_far_$TAG python tools/profile_one.py > gpurun_out/ncu_far_$TAG.log 2>&1
tail -2 gpurun_out/ncu_far_$TAG.log
