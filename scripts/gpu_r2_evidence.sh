# Round-2 evidence in one call: bench line + reference arm, launch list,
# ncu --set full of the trace kernel and of the LiDAR kernel, SASS source page.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH=$? >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
CMD="python bench.py --steps 2 --warmup 3 --latency-calls 5 --no-cpu-baseline --no-parity --no-configs"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
python scripts/profile_target.py > gpurun_out/pt_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 -s 1 -c 1 -f -o gpurun_out/prof_full python scripts/profile_target.py > gpurun_out/ncu_full.log 2>&1
python scripts/profile_lidar.py > gpurun_out/pl_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lidar_warp -s 1 -c 1 -f -o gpurun_out/prof_lidar python scripts/profile_lidar.py > gpurun_out/ncu_lidar.log 2>&1
ncu -i gpurun_out/prof_full.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_full_sass.csv 2>/dev/null; gzip -f gpurun_out/prof_full_sass.csv
NCU_SUMMARY_DIR=gpurun_out python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep 02 > /dev/null 2>&1
NCU_SUMMARY_DIR=gpurun_out python scripts/ncu_summary.py gpurun_out/prof_lidar.ncu-rep 02 lidar > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep  # (64 MiB copy-back limit)
ls -la gpurun_out > gpurun_out/ls.txt
echo DONE
