# threshold / slicing sweep for the class-0 lane kernel (timing only; not a bench line)
for it in 2 4 8; do
  echo "items=$it"; WV_LANE_ITEMS=$it python scripts/variant_sweep.py c2,c3_slice x 15 2>&1 | grep lane2
done
for th in 8388608 33554432 134217728; do
  echo "EG_BIG from $th"; WV_TH_EG_BIG=$th python scripts/variant_sweep.py c3_slice,pin_v x 15 2>&1 | grep lane2
done
echo "BG_BIG from 33554432 (c3_slice_both)"; WV_TH_BG_BIG=33554432 WV_TH_EG_BIG=33554432 python scripts/variant_sweep.py c3_slice_both x 15 2>&1 | grep lane2
python scripts/variant_sweep.py c3_slice_both x 15 2>&1 | grep lane2
