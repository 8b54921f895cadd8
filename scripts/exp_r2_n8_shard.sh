cat > /tmp/one_shard.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, paper_2101_11157_b200 as wv
from paper_2101_11157_b200.workloads import CONFIGS
w = CONFIGS["c2"]; n = int(sys.argv[1]); s = int(sys.argv[2])
ds = wv.DeviceSearch(w.lo, w.hi, w.mode, s, n)
for _ in range(2): ds.run()
torch.cuda.synchronize(); print("ok")
PY
ncu --set full --import-source on --clock-control none -k regex:residue_lane2 -s 1 -c 1 -o gpurun_out/r2_n8s5 python /tmp/one_shard.py 8 5 > /dev/null 2>&1
python scripts/ncu_summary.py rep gpurun_out/r2_n8s5.ncu-rep > gpurun_out/r2_n8s5_residue_kernel_full.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_n8s5_launches.csv python /tmp/one_shard.py 8 5 > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/r2_n8s5_launches.csv > gpurun_out/r2_n8s5_launches.txt
rm -f gpurun_out/r2_n8s5.ncu-rep
