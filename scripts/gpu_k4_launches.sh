mkdir -p gpurun_out
python scripts/profile_k4.py > gpurun_out/k4_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_ray --log-file gpurun_out/k4_launches.csv python scripts/profile_k4.py > /dev/null 2>&1
echo DONE
