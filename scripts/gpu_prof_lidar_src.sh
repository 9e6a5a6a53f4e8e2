mkdir -p gpurun_out
python scripts/profile_lidar.py > gpurun_out/pl_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lidar_warp -s 1 -c 1 -f -o gpurun_out/prof_lidar python scripts/profile_lidar.py > gpurun_out/ncu_lidar.log 2>&1
ncu -i gpurun_out/prof_lidar.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_lidar_sass.csv 2>/dev/null; gzip -f gpurun_out/prof_lidar_sass.csv
ncu -i gpurun_out/prof_lidar.ncu-rep --page details --csv > gpurun_out/prof_lidar_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
echo DONE
