#!/usr/bin/env bash
# One GPU-box pass: parity tests, smoke, bench, launch list and one ncu
# capture of the top kernel.  Run under gpurun from the repo root:
#   gpurun --timeout 1500 -- 'bash tools/gpu_check.sh [tag]'
# Everything lands in gpurun_out/<tag>/.
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1

timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest_gpu exit $?" >> "$OUT/status.txt"

timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke exit $?" >> "$OUT/status.txt"

timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/status.txt"

timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > "$OUT/ncu_launches.log" 2>&1
echo "ncu launches exit $?" >> "$OUT/status.txt"

timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_head_b1 -s 5 -c 2 \
    -o "$OUT/prof_head_b1" python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > "$OUT/ncu_full.log" 2>&1
echo "ncu full exit $?" >> "$OUT/status.txt"

# tensor-core layer GEMM: ncu captures (cfg2 layer 0 at batch 256, cfg4
# dense layer 0 at batch 64), phase timelines, latency by batch, configs
bash tools/run_prof_gemm.sh "$TAG" 256 > /dev/null 2>&1
echo "ncu gemm exit $?" >> "$OUT/status.txt"
timeout 120 python tools/gemm_timeline.py --batch 256 --chunks 24 > "$OUT/gemm_timeline_b256.txt" 2>&1
timeout 120 python tools/gemm_timeline.py --batch 64 --dense --chunks 24 > "$OUT/gemm_timeline_dense.txt" 2>&1
timeout 300 python tools/diag_latency.py --batches 1,2,3,4,8,16,32,64,128,256 > "$OUT/latency_by_batch.txt" 2>&1
timeout 300 python tools/diag_configs.py > "$OUT/configs.txt" 2>&1
[ -x tools/bin/mb_mma ] && timeout 60 ./tools/bin/mb_mma > "$OUT/mb_mma.txt" 2>&1
echo "done" >> "$OUT/status.txt"
