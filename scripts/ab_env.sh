#!/bin/bash
# A/B of environment knobs on the C2 bench (one box): scripts/ab_env.sh "VAR=a" "VAR=b" ...
# prints ms_per_step and the residue kernel's ms for each setting, twice, interleaved.
for rep in 1 2; do
  for kv in "$@"; do
    env $kv python bench.py --steps 10 --no-cpu-baseline --no-e2e --frontier-steps 0 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$kv', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_step'],3))"
  done
done
