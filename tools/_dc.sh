mkdir -p gpurun_out/s4r
for w in 2 3; do
echo "== WST=$w"; SKAN_GEMM_WST=$w timeout 60 python tools/diag_latency.py --batches 4,64,256 --reps 100 2>&1 | grep "flush=True"
done > gpurun_out/s4r/lat.txt
