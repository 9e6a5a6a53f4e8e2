# LiDAR A/B: bash scripts/gpu_lidar_ab.sh name1 name2 ... (librmpb_<name>.so; "default" = librmpb.so)
mkdir -p gpurun_out
: > gpurun_out/lab.jsonl
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; fi
  echo "{\"lib\": \"$v\"}" >> gpurun_out/lab.jsonl
  RMPB_LIBRARY=$lib timeout 300 python scripts/probe_lidar.py 38000 >> gpurun_out/lab.jsonl 2>> gpurun_out/lab.err
done
done
echo DONE
