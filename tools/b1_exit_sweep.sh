#!/usr/bin/env bash
# Event time of the batch-1 kernel when every CTA returns right after phase
# stamp n (SKAN_B1_EXIT_AT): cumulative cost of the phases, launch included.
for n in 100 1 2 3 4 5 7 0; do
  echo "== exit_at $n"
  SKAN_B1_EXIT_AT=$n python tools/diag_latency.py --batches 1 --reps ${REPS:-600} 2>&1 | grep "flush=True"
done
