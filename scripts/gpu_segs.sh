mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for rep in 1 2; do
for sr in 0 8192 16384 65536; do
  SEG_RAYS=$sr timeout 300 python scripts/probe_ab.py >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
done
echo DONE
