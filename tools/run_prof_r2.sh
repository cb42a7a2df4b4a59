#!/usr/bin/env bash
# Round-2 profile pass (one GPU): launch list of the default bench command,
# ncu --set full captures of the batch-1 head kernel, the fp16 int8 layer
# GEMM at batch 256 and the fp16 persistent dense GEMM (cfg4), and the
# phase timelines.  Everything lands in gpurun_out/<tag>/.
set -u
OUT=gpurun_out/${1:-r2prof}; mkdir -p $OUT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
echo "launches $?" >> $OUT/status
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_head_b1 -s 5 -c 1 \
    -o $OUT/prof_head_b1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > $OUT/ncu_b1.log 2>&1
echo "ncu b1 $?" >> $OUT/status
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_layer_gemm" -s 0 -c 1 \
    -o $OUT/prof_gemm_b256 python tools/diag_latency.py --batches 256 --reps 1 > $OUT/ncu_gemm.log 2>&1
echo "ncu gemm $?" >> $OUT/status
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_dense_persist" -s 2 -c 1 \
    -o $OUT/prof_dense python tools/diag_configs.py --only-dense --reps 1 > $OUT/ncu_dense.log 2>&1
echo "ncu dense $?" >> $OUT/status
timeout 120 python tools/b1_timeline.py --reps 2 > $OUT/b1_timeline.txt 2>&1
timeout 120 python tools/gemm_timeline.py --batch 256 --chunks 16 > $OUT/gemm_timeline_b256.txt 2>&1
timeout 120 python tools/dense_timeline.py --chunks 16 > $OUT/dense_timeline.txt 2>&1
timeout 300 python tools/diag_latency.py --batches 1,2,3,4,8,16,32,64,128,256 > $OUT/latency_by_batch.txt 2>&1
timeout 300 python tools/diag_configs.py > $OUT/configs.txt 2>&1
echo "done" >> $OUT/status
