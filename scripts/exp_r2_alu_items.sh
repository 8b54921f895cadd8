set -x
for rep in 1 2; do
for v in 0 1 2 3; do
  if [ $v = 0 ]; then L=""; else L="WV_LIB=paper_2101_11157_b200/ab/libwv_alu$v.so"; fi
  env $L python bench.py --steps 10 --no-cpu-baseline --no-e2e --frontier-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('alu$v', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_per_step'],3))"
done
done
for it in 1 2 3 4 6; do WV_LANE_ITEMS=$it python scripts/shard_timing.py 8 2>&1 | sed "s/^/items=$it /"; done
NS=8 python scripts/shard_breakdown.py 2>&1 | tail -12
