{
for v in default gen4 default gen4; do
if [ $v = default ]; then unset STHK_LIB; else export STHK_LIB=tools/variants/libsthk_$v.so; fi
echo "== $v"; QP_REPS=40 python tools/perf_matrix.py
done
} > gpurun_out/v.txt 2>&1
