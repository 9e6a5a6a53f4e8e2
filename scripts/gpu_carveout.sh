# Shared-memory carveout sweep of the trace kernel on the bench workload.
mkdir -p gpurun_out
for c in default 34 40 50 75 100 default; do
  if [ "$c" = default ]; then CARVEOUT= timeout 300 python scripts/probe_ab.py; else CARVEOUT=$c timeout 300 python scripts/probe_ab.py; fi
done > gpurun_out/carveout.jsonl 2>&1
echo DONE
