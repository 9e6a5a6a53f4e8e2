mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 600 python scripts/bench_configs.py --only c3 > gpurun_out/c3.jsonl 2> gpurun_out/c3.err
timeout 300 python scripts/probe_variants.py > gpurun_out/var_default.log 2>&1
echo DONE
