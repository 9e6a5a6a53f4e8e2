mkdir -p gpurun_out
for lib in librmpb librmpb_nopf; do
RMPB_LIBRARY=$PWD/paper_2301_08068_b200/$lib.so timeout 300 python scripts/probe_lidar.py 3 3:152000 4:24000 4:48000 > gpurun_out/lpf_$lib.json 2>&1
done
echo DONE
