mkdir -p gpurun_out
PROBE_REPS=9 timeout 300 python scripts/probe_ab.py > gpurun_out/q2.jsonl 2> gpurun_out/q2.err
timeout 300 python scripts/probe_lidar.py 38000 50000 >> gpurun_out/q2.jsonl 2>> gpurun_out/q2.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
echo DONE
