# ncu capture of the large-batch layer kernel (one GPU)
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(fwd_large|layer_gemm|split_reduce)" -s 3 -c 3 \
    -o $OUT/prof_large python tools/diag_latency.py --batches 256 --reps 3 > $OUT/ncu_full.log 2>&1
echo "ncu $?" >> $OUT/status
