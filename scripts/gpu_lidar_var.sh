# LiDAR kernel variant sweep: bash scripts/gpu_lidar_var.sh lib1 lib2 ... (default = shipped lib)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; fi
  RMPB_LIBRARY=$lib timeout 300 python scripts/probe_lidar.py 2 3:38000 3:76000 3:152000 > gpurun_out/lvar_$v.json 2>&1
done
echo DONE
