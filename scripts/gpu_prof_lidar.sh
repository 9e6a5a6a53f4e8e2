mkdir -p gpurun_out
python scripts/profile_lidar.py > gpurun_out/pl_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lidar_warp -s 1 -c 1 -o gpurun_out/prof_lidar python scripts/profile_lidar.py > gpurun_out/ncu_lidar.log 2>&1
echo DONE
