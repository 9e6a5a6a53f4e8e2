mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
for v in unroll3 unroll4 u3r12; do
  if [ -z "$v" ]; then lib=""; name=default; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; name=$v; fi
  RMPB_LIBRARY=$lib timeout 300 python scripts/probe_variants.py > gpurun_out/var_$name.log 2>&1
done
echo DONE
