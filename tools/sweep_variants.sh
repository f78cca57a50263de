#!/bin/bash
# Development sweep of kernel knobs (env vars) at the bench shape.
for order in ${ORDERS:-1 0}; do for poly in ${POLYS:-0 2}; do
  echo "== USP_UNIT_ORDER=$order USP_FA_POLY=$poly"
  USP_UNIT_ORDER=$order USP_FA_POLY=$poly timeout 60 python tools/quick_time.py ${LENS:-8192 32768 131072} 2>&1 | grep -v Warn | head -4
done; done
