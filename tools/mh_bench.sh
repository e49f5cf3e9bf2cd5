# BASELINE config 5: reference adaptive MH chain (runChain, verbatim) at N=85k
# C2 data, driven by the B200 engine (full 10,000 iterations) and by the
# reference CPU engine on all host cores (K=20 iterations, extrapolated).
set -e
mkdir -p gpurun_out
LANES=4; grep -q avx512f /proc/cpuinfo && LANES=8
REFX=oracle/_ref/mh_chain_ref_v3; [ $LANES = 8 ] && REFX=oracle/_ref/mh_chain_ref_v4
./oracle/_ref/mh_chain_b200 --n 85000 --data c2 --iters ${ITERS:-10000} --burnin 1000 --seed 1 | tee gpurun_out/mh_b200.json
$REFX --n 85000 --data c2 --iters 20 --burnin 1 --seed 1 --threads 0 --lanes $LANES | tee gpurun_out/mh_ref_cpu.json
