mkdir -p gpurun_out
timeout 700 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
python scripts/profile_target.py > gpurun_out/pt_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 -s 1 -c 2 -o gpurun_out/prof_k2 python scripts/profile_target.py > gpurun_out/ncu_k2.log 2>&1
echo DONE
