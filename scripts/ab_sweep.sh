# A/B of alternative builds (scripts/alt/*.so via WV_LIB) on the class-0 windows (timing only)
for lib in paper_2101_11157_b200/libwv.so scripts/alt/libwv_abel.so; do
  echo "$lib"; WV_LIB=$lib python scripts/variant_sweep.py c2,c3_slice,c3_slice_both x 15 2>&1 | grep lane2
done
