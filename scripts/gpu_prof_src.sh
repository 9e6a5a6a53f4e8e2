# Full ncu capture (with SASS source counters) of one batched k_ray_policy2 launch.
mkdir -p gpurun_out
export PROBE_P=${PROBE_P:-1024}
python scripts/profile_target.py > gpurun_out/pt_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 -s 1 -c 1 -f -o gpurun_out/prof_src python scripts/profile_target.py > gpurun_out/ncu_src.log 2>&1
ncu -i gpurun_out/prof_src.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_src_sass.csv 2> gpurun_out/prof_src_sass.err
echo DONE
