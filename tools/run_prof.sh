# ncu capture of the batch-1 head kernel + its timeline (one GPU)
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 300 python tools/b1_timeline.py --reps 2 > $OUT/timeline.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_head_b1 -s 5 -c 1 \
    -o $OUT/prof_head_b1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
echo "ncu $?" >> $OUT/status
