mkdir -p gpurun_out
(lscpu; nproc; free -g; nvidia-smi; nvidia-smi topo -m) > gpurun_out/host_info.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_fp64.csv &
CP=$!
./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
kill $CP
cat gpurun_out/fp64_peak.json
grep -E "Model name|^CPU\(s\)|Flags" gpurun_out/host_info.txt | cut -c1-200
