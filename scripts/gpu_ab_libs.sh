# A/B of librmpb builds on the bench workload (RMPB_LIBRARY), interleaved
mkdir -p gpurun_out
for rep in 1 2; do
for lib in librmpb.so librmpb_nw4m9.so librmpb_nw4m10.so librmpb_m5.so; do
  RMPB_LIBRARY=$PWD/paper_2301_08068_b200/$lib PROBE_REPS=7 timeout 300 python scripts/probe_ab.py >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done; done
echo DONE
