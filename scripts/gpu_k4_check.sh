bash scripts/gpu_k4_launches.sh
timeout 600 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_server.py -m gpu -q -x > gpurun_out/exs.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bq.json 2>/dev/null
