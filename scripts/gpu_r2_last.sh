# End-of-round evidence: GPU suite (+ the bounds-checked build), smoke, bench
# line + reference arm + C5, launch list, ncu of the trace and LiDAR kernels,
# the config sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest_final.log
RMPB_LIBRARY=$PWD/paper_2301_08068_b200/librmpb_checked.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/checked_pytest.log
RMPB_LIBRARY=$PWD/paper_2301_08068_b200/librmpb_checked.so timeout 600 python scripts/sanitize_suite.py > gpurun_out/checked_suite.log 2>&1; echo RC=$? >> gpurun_out/checked_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE=$? >> gpurun_out/smoke.log
bash scripts/gpu_r2_evidence.sh > gpurun_out/evidence.log 2>&1
timeout 2000 python scripts/bench_configs.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/configs.err
echo DONE
