# K5 DDA: parity test, then the K5 measurement per librmpb build
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dda" > gpurun_out/dda.log 2>&1
: > gpurun_out/k5.jsonl
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; fi
  RMPB_LIBRARY=$lib timeout 300 python scripts/bench_configs.py --only k5 >> gpurun_out/k5.jsonl 2>> gpurun_out/k5.err
done
echo DONE
