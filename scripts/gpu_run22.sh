mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 300 python scripts/probe_variants.py > gpurun_out/var_default.log 2>&1
timeout 300 python scripts/probe_latency.py > gpurun_out/probe.log 2>&1
echo DONE
