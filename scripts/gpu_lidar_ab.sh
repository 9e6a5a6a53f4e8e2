mkdir -p gpurun_out
for lib in librmpb.so librmpb_p3.so librmpb_p6.so librmpb_p8.so; do
  echo "== $lib" >> gpurun_out/lidar_ab.jsonl
  RMPB_LIBRARY=$PWD/paper_2301_08068_b200/$lib timeout 300 python scripts/probe_lidar.py 3:76000 6:76000 6:38000 3:19000 6:19000 6:9500 >> gpurun_out/lidar_ab.jsonl 2>> gpurun_out/lidar_ab.err
done
echo DONE
