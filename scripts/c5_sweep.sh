#!/bin/bash
# Advance the full configs[4] sweep (C5 = [3.9e10, 4.0e10), W+V) on one B200 in checkpointed blocks of 2^22
# integers (paper_2101_11157_b200/sweep.py): resumes from profiles/r2_c5_sweep_state.json if present, stops
# starting new blocks after $1 seconds; the state comes back in gpurun_out/c5_sweep_state.json.
LIMIT=${1:-3600}
mkdir -p gpurun_out
[ -f profiles/r2_c5_sweep_state.json ] && cp profiles/r2_c5_sweep_state.json gpurun_out/c5_sweep_state.json
python - "$LIMIT" <<'PY'
import json, sys, time
sys.path.insert(0, ".")
from paper_2101_11157_b200 import sweep
limit = float(sys.argv[1]); t0 = time.time(); path = "gpurun_out/c5_sweep_state.json"
lo, hi, block = 39 * 10 ** 9, 40 * 10 ** 9, 1 << 22
while time.time() - t0 < limit:
    s = sweep.sweep(lo, hi, 3, block, path, max_blocks=1)
    print(json.dumps({k: s[k] for k in ("next_block", "blocks", "primes", "checksum", "near", "hits", "done")}),
          f"{time.time() - t0:.0f}s", flush=True)
    if s["done"]:
        break
PY
