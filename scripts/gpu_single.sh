mkdir -p gpurun_out
timeout 300 python scripts/probe_single_timeline.py > gpurun_out/single_timeline.jsonl 2> gpurun_out/single_timeline.err
CMD="python scripts/probe_single_timeline.py"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none --csv --log-file gpurun_out/single_launches.csv $CMD > /dev/null 2>&1
echo DONE
