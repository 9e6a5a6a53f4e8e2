# Variant sweep: bash scripts/gpu_var.sh name1 name2 ...  ("" = default lib)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=$PWD/paper_2301_08068_b200/librmpb_$v.so; fi
  RMPB_LIBRARY=$lib timeout 300 python scripts/probe_variants.py > gpurun_out/var_$v.log 2>&1
done
echo DONE
