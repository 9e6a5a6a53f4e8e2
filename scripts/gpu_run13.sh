mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 1500 python scripts/bench_configs.py --oracle-c5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo CONFIGS=$? >> gpurun_out/configs.err
echo DONE
