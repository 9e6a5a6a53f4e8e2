mkdir -p gpurun_out
python scripts/profile_target.py > gpurun_out/pt_plain.log 2>&1 && timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"^k_ray_policy$" -s 1 -c 1 -o gpurun_out/prof_p1 python scripts/profile_target.py > gpurun_out/ncu_p1.log 2>&1
echo DONE
