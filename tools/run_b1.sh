set -u
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest $?" >> $OUT/status
timeout 300 python tools/diag_latency.py --batches 1,2,256 > $OUT/lat.txt 2>&1
timeout 300 python tools/b1_timeline.py --reps 2 > $OUT/timeline.txt 2>&1
[ -x tools/bin/mb_fp64 ] && ./tools/bin/mb_fp64 > $OUT/mb_fp64.txt 2>&1
