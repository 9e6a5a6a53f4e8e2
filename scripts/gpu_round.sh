# Round-end evidence in one call: GPU tests, smoke, bench line, reference arm,
# launch list and one full ncu capture of the hot kernel (summaries: see
# scripts/ncu_summary.py).  Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE=$? >> gpurun_out/smoke.log
bash scripts/gpu_bench.sh
echo DONE
