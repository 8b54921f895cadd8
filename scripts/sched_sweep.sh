# lane-slice sweep for the class-0 lane kernel (timing only; not a bench line)
for it in 2 3 4 5; do
  echo "items=$it"; WV_LANE_ITEMS=$it python scripts/variant_sweep.py c2,c3_slice x 15 2>&1 | grep lane2
done
