# bounds-checked build (stand-in for compute-sanitizer, closed on this pool):
# the whole GPU test-suite and the sanitize workload against librmpb_checked.so
mkdir -p gpurun_out
export RMPB_LIBRARY=$PWD/paper_2301_08068_b200/librmpb_checked.so
timeout 600 python scripts/sanitize_suite.py > gpurun_out/checked_suite.log 2>&1; echo RC=$? >> gpurun_out/checked_suite.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/checked_pytest.log
unset RMPB_LIBRARY
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH=$? >> gpurun_out/bench.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo BENCH=$? >> gpurun_out/bench_c5.err
echo DONE
