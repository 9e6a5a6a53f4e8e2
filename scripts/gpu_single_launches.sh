mkdir -p gpurun_out
for mr in 0.000001 10; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_ray --log-file gpurun_out/single_launch_$mr.csv python scripts/profile_single.py $mr > /dev/null 2>&1
done
echo DONE
