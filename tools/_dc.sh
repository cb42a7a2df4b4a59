mkdir -p gpurun_out/s5a
timeout 120 python tools/gemm_check.py > gpurun_out/s5a/gc.txt 2>&1
for rep in 1 2; do timeout 60 python tools/diag_latency.py --batches 4,64,256 --reps 100 2>&1 | grep "flush=True"; done > gpurun_out/s5a/lat.txt
