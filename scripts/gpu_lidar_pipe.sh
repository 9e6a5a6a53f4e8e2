mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lidar" > gpurun_out/lidar_tests.log 2>&1; echo PYTEST=$? >> gpurun_out/lidar_tests.log
POINT_KERNELS=3,6,7 timeout 300 python scripts/probe_lidar.py 3 6 7/2 7/4 7/8 7/16 7/32 > gpurun_out/lvar_pipe.json 2>&1
echo DONE
