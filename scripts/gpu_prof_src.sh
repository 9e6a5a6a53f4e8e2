# SASS-level ncu source counters of the trace kernel (1024 poses) and of the
# LiDAR warp kernel (v3) on C3; gzipped CSVs in gpurun_out/ (summarise with
# scripts/sass_hot.py).
mkdir -p gpurun_out
export PROBE_P=1024
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 -s 1 -c 1 -f -o gpurun_out/prof_src python scripts/profile_target.py > gpurun_out/ncu_src.log 2>&1
ncu -i gpurun_out/prof_src.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_src_sass.csv 2> gpurun_out/prof_src_sass.err
if [ -z "$NO_LIDAR" ]; then
LIDAR_KERNEL=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lidar -s 1 -c 1 -f -o gpurun_out/prof_lidar python scripts/profile_lidar.py > gpurun_out/ncu_lidar.log 2>&1
ncu -i gpurun_out/prof_lidar.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_lidar_sass.csv 2> gpurun_out/prof_lidar_sass.err
fi
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/*_sass.csv
echo DONE
