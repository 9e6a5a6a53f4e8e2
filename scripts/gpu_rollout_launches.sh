mkdir -p gpurun_out
python scripts/profile_rollout1.py > gpurun_out/r1_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_ray|k_rollout" --log-file gpurun_out/r1_launches.csv python scripts/profile_rollout1.py > /dev/null 2>&1
echo DONE
