# A/B of alternative builds (scripts/alt/*.so via WV_LIB) on the class-1 windows (timing only)
for lib in paper_2101_11157_b200/libwv.so scripts/alt/libwv_f1.so; do
  echo "$lib"; WV_LIB=$lib python scripts/variant_sweep.py x c4_head,c5_head 16,17 2>&1 | grep tuples
done
