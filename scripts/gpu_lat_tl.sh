# Single-pose device timeline: librmpb built with -DRMPB_DBG_TIMELINE (lean
# kernel stamps %globaltimer at CTA start / trace + CTA reduce end / ticket /
# fold / slot written) into paper_2301_08068_b200/dbg/, driven by
# scripts/lat_tl.cu.  Build here:
#   (cd paper_2301_08068_b200/csrc && nvcc <Makefile FLAGS> -shared -DRMPB_DBG_TIMELINE \
#      -o ../dbg/librmpb.so rmpb_api.cu)
#   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -I include scripts/lat_tl.cu \
#      -L paper_2301_08068_b200/dbg -lrmpb -o scripts/lat_tl
mkdir -p gpurun_out
python scripts/probe_lat_c.py
LD_LIBRARY_PATH=$PWD/paper_2301_08068_b200/dbg ./scripts/lat_tl | tee gpurun_out/lat_tl.jsonl
LD_LIBRARY_PATH=$PWD/paper_2301_08068_b200 ./scripts/lat_c | tee gpurun_out/lat_c.jsonl
