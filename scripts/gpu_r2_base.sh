# Round-2 baseline on a fresh box: GPU tests, bench line, SASS source
# counters of the trace kernel and the LiDAR kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH=$? >> gpurun_out/bench.err
bash scripts/gpu_prof_src.sh
echo DONE
