mkdir -p gpurun_out
timeout 600 python scripts/probe_lidar.py 3:76000 6:76000 3:38000 6:38000 6:19000 6:9500 6:150000 > gpurun_out/lidar_r2.jsonl 2> gpurun_out/lidar_r2.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "lidar" > gpurun_out/lidar_tests.log 2>&1; echo RC=$? >> gpurun_out/lidar_tests.log
echo DONE
