# LiDAR kernel variant sweep on C3: bash scripts/gpu_lidar_var.sh lib1 lib2 ...
# (librmpb_<name>.so; "default" = librmpb.so), after the LiDAR parity tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lidar" > gpurun_out/lidar_tests.log 2>&1; echo PYTEST=$? >> gpurun_out/lidar_tests.log
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; fi
  RMPB_LIBRARY=$lib POINT_KERNELS=3,6 timeout 300 python scripts/probe_lidar.py 3 6 6:38000 6:152000 6:19000 > gpurun_out/lvar_$v.json 2>&1
done
echo DONE
