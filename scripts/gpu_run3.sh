mkdir -p gpurun_out
timeout 700 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 300 python scripts/probe_variants.py > gpurun_out/variants_minb4.log 2>&1
RMPB_LIBRARY=$PWD/paper_2301_08068_b200/librmpb_minb3.so timeout 300 python scripts/probe_variants.py > gpurun_out/variants_minb3.log 2>&1
RMPB_LIBRARY=$PWD/paper_2301_08068_b200/librmpb_minb2.so timeout 300 python scripts/probe_variants.py > gpurun_out/variants_minb2.log 2>&1
timeout 300 python scripts/probe_latency.py > gpurun_out/probe.log 2>&1
echo DONE
