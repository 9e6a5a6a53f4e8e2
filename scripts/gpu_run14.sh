mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 600 python scripts/bench_configs.py --only c4loop,c3 > gpurun_out/configs2.jsonl 2> gpurun_out/configs2.err; echo CONFIGS=$? >> gpurun_out/configs2.err
timeout 300 python scripts/probe_latency.py > gpurun_out/probe.log 2>&1
echo DONE
