mkdir -p gpurun_out
python scripts/profile_target.py > gpurun_out/pt_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 -s 1 -c 1 -o gpurun_out/prof_cur python scripts/profile_target.py > gpurun_out/ncu_cur.log 2>&1
echo DONE
