mkdir -p gpurun_out
LIDAR_KERNEL=4 LIDAR_TMA_WARPS=${W:-24000} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lidar -s 1 -c 1 -f -o gpurun_out/prof_ltma python scripts/profile_lidar.py > gpurun_out/ncu_ltma.log 2>&1
ncu -i gpurun_out/prof_ltma.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ltma_sass.csv 2> gpurun_out/prof_ltma_sass.err
ncu -i gpurun_out/prof_ltma.ncu-rep --page details --csv > gpurun_out/prof_ltma_details.csv 2>&1
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/*_sass.csv
echo DONE
