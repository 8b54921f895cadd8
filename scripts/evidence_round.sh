# round-end evidence: full-window runs, ncu captures of the residue kernels, bench + launch list
python scripts/full_window_run.py c3 > gpurun_out/ev_c3.log 2>&1
python scripts/full_window_run.py c5_scale > gpurun_out/ev_c5s.log 2>&1
python scripts/full_window_run.py c4 > gpurun_out/ev_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:residue_lane2 -s 1 -c 1 -o gpurun_out/r1f_c2 python scripts/profile_target.py c2 > gpurun_out/ncu_r1f_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:residue_kernel -s 1 -c 1 -o gpurun_out/r1f_c4s python scripts/profile_target.py c4s > gpurun_out/ncu_r1f_c4s.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:residue_kernel -s 1 -c 1 -o gpurun_out/r1f_c5s python scripts/profile_target.py c5s > gpurun_out/ncu_r1f_c5s.log 2>&1
python bench.py > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r1f.log 2>&1
