# A/B: bash scripts/gpu_ab.sh name1 name2 ... (librmpb_<name>.so; "default" = librmpb.so)
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; fi
  RMPB_LIBRARY=$lib PROBE_REPS=7 timeout 300 python scripts/probe_ab.py >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
done
echo DONE
