# ncu evidence for the bench kernel (run on a GPU box; summaries go to profiles/ via scripts/ncu_summary.py)
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
ncu --set full --import-source on --clock-control none -k regex:residue_lane2 -s 1 -c 1 -o gpurun_out/r1h_c2 python scripts/profile_target.py c2 > gpurun_out/ncu_r1h_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_r1h.log 2>&1
python scripts/shard_timing.py > gpurun_out/shard_r1h.log 2>&1
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
