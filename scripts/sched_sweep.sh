# tier-threshold sweep for the class-0 lane kernel (timing only; not a bench line)
python scripts/variant_sweep.py c2 x 15 2>&1 | grep lane2
for th in 1000000 2000000; do
  echo "EG_MID from $th"; WV_TH_EG_MID=$th python scripts/variant_sweep.py c2 x 15 2>&1 | grep lane2
  echo "BG_MID from $th"; WV_TH_BG_MID=$th python scripts/variant_sweep.py c2 x 15 2>&1 | grep lane2
done
for th in 4194304 8388608; do
  echo "EG_BIG/BG_BIG from $th"; WV_TH_EG_BIG=$th WV_TH_BG_BIG=$th python scripts/variant_sweep.py c3_slice_both x 15 2>&1 | grep lane2
done
