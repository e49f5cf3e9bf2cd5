# one full ncu capture of the hot pair kernel (C2, Theta_post) + the raw page as csv
TAG=${TAG:-r01}
ncu --set full --clock-control none --import-source on -k regex:"sym_kernel|pair_kernel" -s 3 -c 1 -o gpurun_out/prof_pair_$TAG python tools/profile_one.py > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
ls -la gpurun_out | grep $TAG
