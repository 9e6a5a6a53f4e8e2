# GPU suite + smoke + the round-2 evidence (bench line, reference arm, C5,
# launch list, ncu of the trace and LiDAR kernels) in one call.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE=$? >> gpurun_out/smoke.log
bash scripts/gpu_r2_evidence.sh > gpurun_out/evidence.log 2>&1
echo DONE
