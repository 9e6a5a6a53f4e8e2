mkdir -p gpurun_out
PROBE_REPS=9 timeout 300 python scripts/probe_ab.py > gpurun_out/qab.jsonl 2> gpurun_out/qab.err
timeout 300 python scripts/probe_lidar.py 76000 38000 19000 >> gpurun_out/qab.jsonl 2>> gpurun_out/qab.err
echo DONE
