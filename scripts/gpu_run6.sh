mkdir -p gpurun_out
./scripts/microbench > gpurun_out/microbench.log 2>&1
timeout 300 python scripts/probe_latency.py > gpurun_out/probe.log 2>&1
echo DONE
