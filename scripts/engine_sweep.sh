#!/bin/bash
# Time windows under each run engine (WV_ENGINE0: class p<2^30, WV_ENGINE1: 2^30<=p<2^44; 0=IMAD 1=FP64 2=mixed)
set -e
for e0 in 0 1 2; do WV_ENGINE0=$e0 python scripts/quick_timing.py c2 pin_v | sed "s/^/E0=$e0 /"; done
for e1 in 0 1 2; do WV_ENGINE1=$e1 python scripts/quick_timing.py c4_head c5_head | sed "s/^/E1=$e1 /"; done
