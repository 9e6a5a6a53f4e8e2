# Standard measurement: bench line, launch list, one full ncu capture of the
# hot kernel.  Outputs land in gpurun_out/ (copy summaries into profiles/).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH=$? >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --latency-calls 5 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
python scripts/profile_target.py > gpurun_out/pt_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 -s 1 -c 1 -o gpurun_out/prof_full python scripts/profile_target.py > gpurun_out/ncu_full.log 2>&1
echo DONE
