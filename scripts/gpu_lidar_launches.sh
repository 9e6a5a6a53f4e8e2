# Per-kernel durations (ncu launch list) of the LiDAR path on C3 for the given kernel options
mkdir -p gpurun_out
for k in "$@"; do
LIDAR_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_lidar --log-file gpurun_out/lidar_launch_k$k.csv python scripts/profile_lidar.py > /dev/null 2>&1
done
echo DONE
