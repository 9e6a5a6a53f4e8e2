mkdir -p gpurun_out
python scripts/profile_pinv_cost.py > gpurun_out/pc_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_ray --log-file gpurun_out/pc_launches.csv python scripts/profile_pinv_cost.py > /dev/null 2>&1
echo DONE
