{
for i in 1 2 3; do for g in 1 0; do
echo "== STHK_GRAPH=$g run $i"
STHK_GRAPH=$g ./oracle/_ref/mh_chain_b200 --n 85000 --data c2 --iters 10000 --burnin 1000 --seed 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['seconds'])"
done; done
STHK_GRAPH=1 ./tools/call_latency 85000
nproc; cat /proc/cpuinfo | grep "model name" | head -1
} > gpurun_out/mh3.txt 2>&1
