#!/usr/bin/env bash
# cfg4 dense step time across persistent-kernel knobs (L2 prefetch distance)
for d in ${DISTS:-0 8 16}; do
  echo "== SKAN_DENSE_PREFETCH=$d"; SKAN_DENSE_PREFETCH=$d timeout 300 python tools/diag_configs.py --only-dense 2>&1 | grep cfg4
done
echo "== split GEMM"; SKAN_DENSE_PERSIST=0 timeout 300 python tools/diag_configs.py --only-dense 2>&1 | grep cfg4
