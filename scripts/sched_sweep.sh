# chain-mode / W step-width sweep for the class-0 lane kernel (timing only; not a bench line)
for cm in 1 5; do
  echo "WV_LANE_CHAIN=$cm"; WV_LANE_CHAIN=$cm python scripts/variant_sweep.py c2,c3_slice_both x 15 2>&1 | grep lane2
done
