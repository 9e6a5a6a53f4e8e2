# A/B of the map's L2 access-policy window on the bench workload + device limits
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
python -c "
from cuda.bindings import runtime as rt
for a in ('cudaDevAttrMaxPersistingL2CacheSize','cudaDevAttrMaxAccessPolicyWindowSize','cudaDevAttrL2CacheSize'):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
" > gpurun_out/l2attrs.txt 2>&1
for rep in 1 2; do
for w in 0 1; do
  L2_WINDOW=$w timeout 300 python scripts/probe_ab.py >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
done
echo DONE
