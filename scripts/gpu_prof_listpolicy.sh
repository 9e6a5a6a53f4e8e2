mkdir -p gpurun_out
LIDAR_KERNEL=6 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lidar_listpolicy -s 1 -c 1 -f -o gpurun_out/prof_lp python scripts/profile_lidar.py > gpurun_out/ncu_lp.log 2>&1
ncu -i gpurun_out/prof_lp.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_lp_sass.csv 2> /dev/null
ncu -i gpurun_out/prof_lp.ncu-rep --page details --csv > gpurun_out/prof_lp_details.csv 2> /dev/null
rm -f gpurun_out/*.ncu-rep; gzip -f gpurun_out/prof_lp_sass.csv
echo DONE
