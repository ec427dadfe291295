#!/bin/bash
# pageable host -> GPU through the pacer's ring: workers x ring size (each twice)
for w in ${WORKERS:-4 8 12 16}; do for r in ${RINGS:-20000000 40000000 80000000}; do for rep in 1 2; do
  echo "workers=$w ring=$r $(FT_PACER_WORKERS=$w FT_HOST_RING_BYTES=$r timeout 120 python tools/diag_pageable.py 2>&1 | grep pageable)"
done; done; done
