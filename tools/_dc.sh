mkdir -p gpurun_out/s4j
timeout 120 python tools/dense_check.py > gpurun_out/s4j/dc.txt 2>&1; echo "rc $?" >> gpurun_out/s4j/dc.txt
timeout 60 python tools/dense_timeline.py --chunks 10 > gpurun_out/s4j/tl.txt 2>&1
for rep in 1 2; do
echo "== f16"; timeout 60 python tools/diag_configs.py --only-dense 2>&1 | grep cfg4
echo "== tf32"; SKAN_DENSE_F16=0 timeout 60 python tools/diag_configs.py --only-dense 2>&1 | grep cfg4
done > gpurun_out/s4j/sweep.txt
