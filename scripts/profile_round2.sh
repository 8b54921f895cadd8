#!/bin/bash
# Round-2 evidence on one B200 (run from the repo root under gpurun); outputs in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --frontier-steps 0 > gpurun_out/r2_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:residue_lane2 -s 1 -c 1 -o gpurun_out/r2_c2 \
    python scripts/profile_target.py c2 > gpurun_out/r2_ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:residue_kernel -s 1 -c 1 -o gpurun_out/r2_c5s \
    python scripts/profile_target.py c5s > gpurun_out/r2_ncu_c5s.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:Mont64, \(int\)2, \(int\)0, \(int\)8" -s 1 -c 1 -o gpurun_out/r2_c2big \
    python scripts/profile_target.py c2big > gpurun_out/r2_ncu_c2big.log 2>&1
python scripts/shard_timing.py > gpurun_out/r2_shard.log 2>&1
python scripts/full_window_run.py c4 > gpurun_out/r2_full_c4.log 2>&1
# summaries on the box (gpurun_out/ comes back only under 64 MiB): keep the C2 report, summarise the others
for t in c2 c5s c2big; do python scripts/ncu_summary.py rep gpurun_out/r2_$t.ncu-rep > gpurun_out/r2_${t}_residue_kernel_full.txt 2>&1; done
python scripts/ncu_summary.py launches gpurun_out/r2_launches.csv > gpurun_out/r2_c2_launches.txt 2>&1
rm -f gpurun_out/r2_c5s.ncu-rep gpurun_out/r2_c2big.ncu-rep
echo done
