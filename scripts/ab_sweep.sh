# A/B of alternative builds (scripts/alt/*.so via WV_LIB) on the class-0 windows (timing only)
for lib in scripts/alt/libwv_w4v4.so scripts/alt/libwv_w6v4.so scripts/alt/libwv_w4v6.so scripts/alt/libwv_w6v6.so scripts/alt/libwv_w5v5.so; do
  echo "$lib"; WV_LIB=$lib python scripts/variant_sweep.py c2,c3_slice,c3_slice_both x 15 2>&1 | grep lane2
done
