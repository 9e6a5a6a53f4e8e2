# LiDAR TMA kernel check: parity tests for every variant, then the C3 sweep.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lidar" > gpurun_out/lidar_tests.log 2>&1; echo PYTEST=$? >> gpurun_out/lidar_tests.log
timeout 300 python scripts/probe_lidar.py 3 4:4000 4:8000 4:12000 4:24000 5:8000 5:12000 > gpurun_out/lidar_tma.json 2> gpurun_out/lidar_tma.err
echo DONE
