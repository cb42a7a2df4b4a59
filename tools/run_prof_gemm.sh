# ncu captures of the tensor-core layer GEMM (one GPU): compressed cfg2 head
# layer 0 at batch 64 and 256, dense cfg4 layer 0 at batch 64
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
for B in ${2:-64 256}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_layer_gemm" -s 0 -c 1 \
    -o $OUT/prof_gemm_b$B python tools/diag_latency.py --batches $B --reps 1 > $OUT/ncu_b$B.log 2>&1
done
if [ -z "${3:-}" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_layer_gemm" -s 2 -c 1 \
    -o $OUT/prof_gemm_dense python tools/diag_configs.py --only-dense --reps 1 > $OUT/ncu_dense.log 2>&1
fi
echo "ncu $?" >> $OUT/status
