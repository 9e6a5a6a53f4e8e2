# ncu source counters of the single-pose (lean) kernel at max range ~0 (fixed
# cost only) and 10 m; gzipped SASS CSVs in gpurun_out/.
mkdir -p gpurun_out
for mr in 0.000001 10; do
python scripts/profile_single.py $mr > gpurun_out/ps_$mr.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy -s 3 -c 1 -f -o gpurun_out/prof_single_$mr python scripts/profile_single.py $mr > gpurun_out/ncu_single_$mr.log 2>&1
ncu -i gpurun_out/prof_single_$mr.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_single_${mr}_sass.csv 2>/dev/null
ncu -i gpurun_out/prof_single_$mr.ncu-rep --page details --csv > gpurun_out/prof_single_${mr}_details.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep; gzip -f gpurun_out/prof_single_*_sass.csv
echo DONE
