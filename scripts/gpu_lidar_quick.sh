mkdir -p gpurun_out
timeout 300 python scripts/probe_lidar.py 38000 50000 76000 25000 > gpurun_out/lq.jsonl 2> gpurun_out/lq.err
timeout 600 python -m pytest tests -m gpu -q -k "lidar or sanit" > gpurun_out/lq_tests.log 2>&1; echo RC=$? >> gpurun_out/lq_tests.log
echo DONE
timeout 300 python scripts/sanitize_suite.py > gpurun_out/lq_suite.log 2>&1; echo RC=$? >> gpurun_out/lq_suite.log
